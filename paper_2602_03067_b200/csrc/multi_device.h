// Multi-GPU sinkhorn_solve inside the library (multi_device.cpp).
#pragma once

#include <vector>

#include "../../include/fsk_b200.h"

namespace fskb {

// fsk_set_num_devices setting: 0 = single-device path, N >= 1 = shard over 0..N-1
int num_devices_setting();

// Runs the alternating solve sharded over the configured devices; false when the
// setting or the schedule does not apply (the caller then runs the single-device
// path). alpha / beta: the potential shifts; f_init / g_init nullable (warm start).
template <typename T>
bool solve_multi_device(const fsk_measure& src, const fsk_measure& tgt, const fsk_cost* cost,
                        const fsk_config& cfg, const std::vector<double>& schedule,
                        const std::vector<double>& alpha, const std::vector<double>& beta,
                        const double* f_init, const double* g_init, const fsk_tiles& tiles,
                        fsk_ledger* ledger, fsk_report* rep, double* grad_out);

}  // namespace fskb
