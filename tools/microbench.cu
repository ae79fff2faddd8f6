// Pipe-rate microbenchmarks on the B200 (sm_100a): MUFU ex2 (f32, f16x2),
// FFMA, and tcgen05.ld TMEM->register bandwidth. Used to size the
// split-fp16 half-step epilogue. Prints per-SM per-clock rates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_ex2(float* out, int iters, long long* cyc) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2h2(float* out, int iters, long long* cyc) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.01f * i, -0.02f); v[i] = *reinterpret_cast<uint32_t*>(&h); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= v[i];
    if (s == 12345u) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma(float* out, int iters, long long* cyc) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = 0.001f * (threadIdx.x + i);
    float a = 0.999f, b = 0.0001f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaf(v[i], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// TMEM: allocate 512 columns, each warp repeatedly loads 32 lanes x 64 cols.
__global__ void k_tmem(float* out, int iters, long long* cyc) {
    __shared__ uint32_t tbase;
    int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t base = tbase;
    uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t col0 = (warp / 4) * 256;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
        uint32_t addr = base + lane_base + col0 + (it & 3) * 32;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
    }
    long long t1 = clock64();
    if (acc == 12345.f) out[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out; long long* cyc; CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&cyc, 148 * 8));
    long long h[148];
    int iters = 4096;
    for (int warps : {4, 8, 16}) {
        int thr = warps * 32;
        k_ex2<<<148, thr>>>(out, iters, cyc); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost));
        printf("ex2.f32   warps=%2d : %.2f ops/clk/SM\n", warps, double(thr) * 8 * iters / h[0]);
        k_ex2h2<<<148, thr>>>(out, iters, cyc); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost));
        printf("ex2.f16x2 warps=%2d : %.2f elem/clk/SM\n", warps, double(thr) * 16 * iters / h[0]);
        k_ffma<<<148, thr>>>(out, iters, cyc); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost));
        printf("ffma      warps=%2d : %.2f ops/clk/SM\n", warps, double(thr) * 8 * iters / h[0]);
    }
    for (int warps : {4, 8}) {
        int thr = warps * 32;
        k_tmem<<<148, thr>>>(out, 2048, cyc); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost));
        printf("tcgen05.ld x32 warps=%d : %.1f bytes/clk/SM\n", warps, double(thr) * 32 * 4 * 2048 / h[0]);
    }
    return 0;
}
