// fsk::set_num_devices - extension of the drop-in (the reference is CPU-only; its
// analogue is set_num_threads, threads.hpp:12-13): how many GPUs of this process
// fsk::solver::sinkhorn_solve shards over. 0 (default) runs on the
// current device; n >= 1 shards rows over devices 0..n-1 with NCCL all-gathers.
#pragma once

namespace fsk {

void set_num_devices(int n);
int num_devices();

}  // namespace fsk
