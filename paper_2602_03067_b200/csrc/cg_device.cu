// Device CG vector algebra (cg_device.h). Reductions: kRedBlocks fixed blocks,
// grid-stride accumulation in a fixed order, a shared-memory tree per block,
// then one block sums the partials in index order.
#include "cg_device.h"

namespace fskb {
namespace {

constexpr int kRedBlocks = 296;   // 2 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[kRedThreads];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    return sh[0];
}

__global__ void finish_sum_kernel(const double* __restrict__ partial, double* __restrict__ out) {
    double v = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) v += partial[i];
    v = block_sum(v);
    if (threadIdx.x == 0) *out = v;
}

__global__ void cg_init_kernel(const double* __restrict__ rhs, int64_t m, double* __restrict__ w2,
                               double* __restrict__ res, double* __restrict__ pdir,
                               float* __restrict__ pf, double* __restrict__ partial) {
    double acc = 0.0;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < m;
         j += int64_t(gridDim.x) * blockDim.x) {
        const double v = rhs[j];
        w2[j] = 0.0;
        res[j] = v;
        pdir[j] = v;
        pf[j] = float(v);
        acc += v * v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void cg_div_rows_kernel(const double* __restrict__ pv, const float* __restrict__ r,
                                   int64_t n, float* __restrict__ out) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = float(pv[i] / double(r[i]));
}

// Ap = c p - ptq + tau p, partial <p, Ap>
__global__ void cg_ap_kernel(const float* __restrict__ c, const double* __restrict__ pdir,
                             const double* __restrict__ ptq, double tau, int64_t m,
                             double* __restrict__ ap, double* __restrict__ partial) {
    double acc = 0.0;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < m;
         j += int64_t(gridDim.x) * blockDim.x) {
        const double p = pdir[j];
        const double v = double(c[j]) * p - ptq[j] + tau * p;
        ap[j] = v;
        acc += p * v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// alpha = rs / pAp; w2 += alpha p; res -= alpha Ap; partial <res, res>
__global__ void cg_update_kernel(const double* __restrict__ rs, const double* __restrict__ pap,
                                 const double* __restrict__ pdir, const double* __restrict__ ap,
                                 int64_t m, double* __restrict__ w2, double* __restrict__ res,
                                 double* __restrict__ partial) {
    const double alpha = *rs / *pap;
    double acc = 0.0;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < m;
         j += int64_t(gridDim.x) * blockDim.x) {
        w2[j] += alpha * pdir[j];
        const double r = res[j] - alpha * ap[j];
        res[j] = r;
        acc += r * r;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void cg_dir_kernel(const double* __restrict__ rs_old, const double* __restrict__ rs_new,
                              const double* __restrict__ res, int64_t m, double* __restrict__ pdir,
                              float* __restrict__ pf) {
    const double beta = *rs_new / *rs_old;
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j < m) {
        const double p = res[j] + beta * pdir[j];
        pdir[j] = p;
        pf[j] = float(p);
    }
}

unsigned blocks_of(int64_t n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

DeviceCg::DeviceCg(int64_t m_, cudaStream_t s_) : m(m_), s(s_) {
    w2.alloc(size_t(m), s);
    res.alloc(size_t(m), s);
    pdir.alloc(size_t(m), s);
    ap.alloc(size_t(m), s);
    pf.alloc(size_t(m), s);
    partial.alloc(kRedBlocks, s);
    scal.alloc(4, s);
    FSKB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h_rs), sizeof(double)));
}

DeviceCg::~DeviceCg() {
    if (h_rs) {
        cudaStreamSynchronize(s);
        cudaFreeHost(h_rs);
    }
}

double DeviceCg::init(const double* rhs_dev) {
    k = 0;
    cg_init_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(rhs_dev, m, w2.get(), res.get(), pdir.get(),
                                                      pf.get(), partial.get());
    finish_sum_kernel<<<1, kRedThreads, 0, s>>>(partial.get(), scal.get() + 0);
    FSKB_CUDA(cudaGetLastError());
    count_launch(2);
    FSKB_CUDA(cudaMemcpyAsync(h_rs, scal.get() + 0, sizeof(double), cudaMemcpyDeviceToHost, s));
    FSKB_CUDA(cudaStreamSynchronize(s));
    return *h_rs;
}

void DeviceCg::div_rows(const double* pv, const float* r, int64_t n, float* tmpf) {
    if (!n) return;
    cg_div_rows_kernel<<<blocks_of(n, 256), 256, 0, s>>>(pv, r, n, tmpf);
    FSKB_CUDA(cudaGetLastError());
    count_launch();
}

double DeviceCg::step(const float* c, const double* ptq, double tau) {
    double* rs = scal.get() + (k & 1);
    double* rs_new = scal.get() + ((k + 1) & 1);
    double* pap = scal.get() + 2;
    cg_ap_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(c, pdir.get(), ptq, tau, m, ap.get(),
                                                    partial.get());
    finish_sum_kernel<<<1, kRedThreads, 0, s>>>(partial.get(), pap);
    cg_update_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(rs, pap, pdir.get(), ap.get(), m, w2.get(),
                                                        res.get(), partial.get());
    finish_sum_kernel<<<1, kRedThreads, 0, s>>>(partial.get(), rs_new);
    FSKB_CUDA(cudaGetLastError());
    count_launch(4);
    FSKB_CUDA(cudaMemcpyAsync(h_rs, rs_new, sizeof(double), cudaMemcpyDeviceToHost, s));
    FSKB_CUDA(cudaStreamSynchronize(s));
    return *h_rs;
}

void DeviceCg::direction() {
    const double* rs = scal.get() + (k & 1);
    const double* rs_new = scal.get() + ((k + 1) & 1);
    cg_dir_kernel<<<blocks_of(m, 256), 256, 0, s>>>(rs, rs_new, res.get(), m, pdir.get(), pf.get());
    FSKB_CUDA(cudaGetLastError());
    count_launch();
    ++k;
}

}  // namespace fskb
