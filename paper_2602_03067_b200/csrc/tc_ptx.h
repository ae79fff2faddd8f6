// Thin inline-PTX layer for the sm_100a kernels: mbarriers, bulk copies (the
// TMA engine's non-tensor path), tcgen05 MMA / TMEM load-store, UMMA
// descriptors, and the tile-image geometry shared by every tcgen05 kernel.
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace fskb {
namespace tc {

constexpr int TILE = 128;                 // rows per query tile / keys per key tile
constexpr int DPAD = 64;                  // padded feature dim (one SW128 chunk)
constexpr uint32_t CHUNK = TILE * 128;    // 16 KB: 128 rows x 64 fp16
constexpr uint32_t QTILE = 2 * CHUNK;     // hi + lo
constexpr uint32_t BIAS = TILE * 32;      // 4 KB: 128 rows x 16 fp16 (SW32)
constexpr uint32_t KSTAGE = 2 * CHUNK + BIAS;  // 36 KB
constexpr float kOnesW0 = 2048.0f, kOnesW2 = 1.0f / 2048.0f;

// idesc, kind::f16, D f32 (bits 4-5 = 1), A/B f16 (0), A K-major.
//   score GEMM  S = Q K^T : B K-major, N = 128, M = 128
//   value GEMM  O = P V   : A from TMEM, B MN-major (bit 16), N = 64, M = 128
constexpr uint32_t IDESC_QK = (1u << 4) | (uint32_t(TILE >> 3) << 17) | (uint32_t(TILE >> 4) << 24);
constexpr uint32_t IDESC_PV =
    (1u << 4) | (1u << 16) | (uint32_t(DPAD >> 3) << 17) | (uint32_t(TILE >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#ifdef FSKB_HANG_DEBUG
    // debug builds: report the barrier a warp is stuck on, then trap
    for (long long i = 0;; ++i) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (i == (1ll << 21) && (threadIdx.x & 31) == 0)
            printf("[hang] block %d thread %d bar 0x%x parity %u\n", int(blockIdx.x),
                   int(threadIdx.x), bar, parity);
        if (i == (1ll << 23)) asm volatile("trap;");
    }
#endif
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor. layout 2 = SWIZZLE_128B, 6 = SWIZZLE_32B;
// version 1. K-major swizzled: SBO = 8-row group stride, LBO unused.
// MN-major SW128: SBO = stride between 8-row K groups, LBO = stride between
// 64-element MN atoms (unused when N = 64).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo, uint32_t layout,
                                              uint32_t lbo = 16) {
    uint64_t d = uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout) << 61;
    return d;
}

// D[tmem] (+)= A[smem] B[smem]. ELECT: called by a converged warp, one elected lane
// issues (no per-instruction divergence handling around the uniform operands)
template <bool ELECT = false>
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
    if constexpr (ELECT)
        asm volatile(
            "{\n"
            ".reg .pred p, e;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(d_tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// D[tmem] (+)= A[tmem] B[smem]
template <bool ELECT = false>
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                        uint32_t idesc, uint32_t acc) {
    const uint32_t z = 0;
    if constexpr (ELECT)
        asm volatile(
            "{\n"
            ".reg .pred p, e;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n"
            "}\n" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(z));
    else
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n"
            "}\n" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc), "r"(z));
}
template <bool ELECT = false>
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    if constexpr (ELECT)
        asm volatile(
            "{\n"
            ".reg .pred e;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
            "}\n" ::"r"(bar)
            : "memory");
    else
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
            : "memory");
}

#define FSKB_TMEM_LD32(addr, r)                                                                  \
    asm volatile(                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),             \
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),          \
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),          \
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),          \
          "=r"(r[31])                                                                            \
        : "r"(addr))

#define FSKB_TMEM_ST32(addr, r)                                                                  \
    asm volatile(                                                                                \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"  \
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::   \
            "r"(addr),                                                                           \
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),        \
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),      \
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),      \
        "r"(r[29]), "r"(r[30]), "r"(r[31])                                                       \
        : "memory")

__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA / ALU pipes (the MUFU unit is the bottleneck of the LSE epilogue
// when few tiles can be skipped): x = n + f, n = rint(x) by the 1.5 * 2^23 magic
// add, f in [-1/2, 1/2], degree-6 minimax polynomial (max relative error 9.6e-8
// with fp32 Horner, vs ~2^-22 for ex2.approx), 2^n added into the exponent field.
// x is clamped at -125 (2^-125 is far below anything an fp32 sum can register).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;
    const float n = t - 12582912.0f;
    const float f = x - n;
    float p = 1.5394332876894623e-4f;
    p = fmaf(p, f, 1.3388522202149034e-3f);
    p = fmaf(p, f, 9.618211537599564e-3f);
    p = fmaf(p, f, 5.550358444452286e-2f);
    p = fmaf(p, f, 2.4022650718688965e-1f);
    p = fmaf(p, f, 6.931471824645996e-1f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Constant "ones" chunk of the query operand, [2048, 1, 1/2048, 0...] per row
// (SW32 K-major): multiplies the 3-piece key bias chunk into the score GEMM.
__device__ __forceinline__ void fill_ones_chunk(uint8_t* dst, int tid, int nthreads) {
    for (int idx = tid; idx < TILE * 16; idx += nthreads) {
        const int r = idx >> 4, k = idx & 15;
        const float v = k == 0 ? kOnesW0 : (k == 1 ? 1.0f : (k == 2 ? kOnesW2 : 0.0f));
        const uint32_t off = r * 32 + ((((k >> 3) ^ ((r >> 2) & 1))) << 4) + (k & 7) * 2;
        *reinterpret_cast<__half*>(dst + off) = __float2half_rn(v);
    }
}

// Issues the 13 MMAs of one split-fp16 score tile: 3 products x 4 K16 slices of
// the 64-wide hi/lo chunks, plus the bias K16 slice. Order matters for the fp32
// accumulator's rounding: the 8 small cross terms (2^-11 of the score) first,
// then the bias, then the 4 hi x hi slices, so only 5 additions round at the
// score's full magnitude and the bias partially cancels the dot product early.
template <bool ELECT = false>
__device__ __forceinline__ void issue_score_tile(uint32_t d_tmem, uint32_t qa, uint32_t ones,
                                                 uint32_t kst) {
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk) {
        const uint64_t ah = umma_desc(qa + kk * 32, 1024, 2);
        const uint64_t al = umma_desc(qa + CHUNK + kk * 32, 1024, 2);
        const uint64_t bh = umma_desc(kst + kk * 32, 1024, 2);
        const uint64_t bl = umma_desc(kst + CHUNK + kk * 32, 1024, 2);
        umma_ss<ELECT>(d_tmem, al, bh, IDESC_QK, kk > 0 ? 1u : 0u);
        umma_ss<ELECT>(d_tmem, ah, bl, IDESC_QK, 1u);
    }
    umma_ss<ELECT>(d_tmem, umma_desc(ones, 256, 6), umma_desc(kst + QTILE, 256, 6), IDESC_QK, 1u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ss<ELECT>(d_tmem, umma_desc(qa + kk * 32, 1024, 2), umma_desc(kst + kk * 32, 1024, 2),
                IDESC_QK, 1u);
}

// Score tile with the query operand in TMEM (A from TMEM at column q: hi at +0,
// lo at +32, ones at +64; 8 columns per K16 slice), same 13-MMA order as above.
template <bool ELECT = false>
__device__ __forceinline__ void issue_score_tile_tq(uint32_t d_tmem, uint32_t q, uint32_t kst) {
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk) {
        umma_ts<ELECT>(d_tmem, q + 32 + kk * 8, umma_desc(kst + kk * 32, 1024, 2), IDESC_QK,
                kk > 0 ? 1u : 0u);
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kst + CHUNK + kk * 32, 1024, 2), IDESC_QK, 1u);
    }
    umma_ts<ELECT>(d_tmem, q + 64, umma_desc(kst + QTILE, 256, 6), IDESC_QK, 1u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kst + kk * 32, 1024, 2), IDESC_QK, 1u);
}
// Half-width (N = 64) forms: keys [64 h, 64 h + 64) of the staged key tile into a
// 64-column accumulator. A query tile then owns two half accumulators, so the MMAs
// of one half overlap the epilogue of the other even when only one query tile of
// the pair is live (the common case of a warm pass).
constexpr uint32_t IDESC_QK64 = (1u << 4) | (uint32_t(64 >> 3) << 17) | (uint32_t(TILE >> 4) << 24);
constexpr uint32_t kHalfK = 64 * 128;   // 64 key rows of a SW128 hi / lo chunk
constexpr uint32_t kHalfB = 64 * 32;    // 64 key rows of the SW32 bias chunk
// Lean issue of a (query tile, 64-key half) chain from a converged warp: one
// elect.sync for the whole chain and the B descriptors derived from one low word by
// 32-bit adds (K-major SW128, LBO 16 B: the low word is (addr >> 4) | 1 << 16, and the
// chain's offsets - 32 B per K16 slice, the 16 KB lo chunk - stay inside its 14-bit
// address field for any shared-memory address < 256 KB). The MMA warp otherwise spends
// ~9 instructions per MMA (descriptor packing, per-instruction elect), which bounds
// the short chains of the screen and warm passes. Same MMAs in the same order.
constexpr uint32_t kDescHiSw128 = (1024u >> 4) | (1u << 14) | (2u << 29);
constexpr uint32_t kDescHiBias = (256u >> 4) | (1u << 14) | (6u << 29);
__device__ __forceinline__ uint32_t desc_lo(uint32_t saddr) {
    return ((saddr & 0x3FFFFu) >> 4) | (1u << 16);
}
// screen: bias (overwrite), then the 4 hi x hi K16 slices
__device__ __forceinline__ void issue_screen_half_lean(uint32_t d, uint32_t q, uint32_t klo,
                                                       uint32_t blo) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b32 a1, a2, a3, ab, k1, k2, k3;\n"
        ".reg .b64 b0, b1, b2, b3, bb;\n"
        "setp.ne.b32 pf, %7, %7;\n"
        "setp.eq.b32 pt, %7, %7;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u32 ab, %1, 64;\n"
        "add.u32 k1, %2, 2;\n"
        "add.u32 k2, %2, 4;\n"
        "add.u32 k3, %2, 6;\n"
        "mov.b64 b0, {%2, %5};\n"
        "mov.b64 b1, {k1, %5};\n"
        "mov.b64 b2, {k2, %5};\n"
        "mov.b64 b3, {k3, %5};\n"
        "mov.b64 bb, {%3, %6};\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ab], bb, %4, {%7, %7, %7, %7}, pf;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %4, {%7, %7, %7, %7}, pt;\n"
        "}\n" ::"r"(d),
        "r"(q), "r"(klo), "r"(blo), "r"(IDESC_QK64), "r"(kDescHiSw128), "r"(kDescHiBias), "r"(0u));
}
__device__ __forceinline__ void issue_screen_half_lean_commit(uint32_t d, uint32_t q, uint32_t klo,
                                                       uint32_t blo, uint32_t bar) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b32 a1, a2, a3, ab, k1, k2, k3;\n"
        ".reg .b64 b0, b1, b2, b3, bb;\n"
        "setp.ne.b32 pf, %7, %7;\n"
        "setp.eq.b32 pt, %7, %7;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u32 ab, %1, 64;\n"
        "add.u32 k1, %2, 2;\n"
        "add.u32 k2, %2, 4;\n"
        "add.u32 k3, %2, 6;\n"
        "mov.b64 b0, {%2, %5};\n"
        "mov.b64 b1, {k1, %5};\n"
        "mov.b64 b2, {k2, %5};\n"
        "mov.b64 b3, {k3, %5};\n"
        "mov.b64 bb, {%3, %6};\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ab], bb, %4, {%7, %7, %7, %7}, pf;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
        "}\n" ::"r"(d),
        "r"(q), "r"(klo), "r"(blo), "r"(IDESC_QK64), "r"(kDescHiSw128), "r"(kDescHiBias), "r"(0u), "r"(bar)
        : "memory");
}
// split-fp16 score: 8 cross terms (lo x hi, hi x lo per K16 slice; the first
// overwrites), bias, 4 hi x hi
__device__ __forceinline__ void issue_score_half_lean(uint32_t d, uint32_t q, uint32_t klo,
                                                      uint32_t blo) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b32 a1, a2, a3, l0, l1, l2, l3, ab, k1, k2, k3, m0, m1, m2, m3;\n"
        ".reg .b64 h0, h1, h2, h3, w0, w1, w2, w3, bb;\n"
        "setp.ne.b32 pf, %7, %7;\n"
        "setp.eq.b32 pt, %7, %7;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u32 l0, %1, 32;\n"
        "add.u32 l1, %1, 40;\n"
        "add.u32 l2, %1, 48;\n"
        "add.u32 l3, %1, 56;\n"
        "add.u32 ab, %1, 64;\n"
        "add.u32 k1, %2, 2;\n"
        "add.u32 k2, %2, 4;\n"
        "add.u32 k3, %2, 6;\n"
        "add.u32 m0, %2, 1024;\n"
        "add.u32 m1, %2, 1026;\n"
        "add.u32 m2, %2, 1028;\n"
        "add.u32 m3, %2, 1030;\n"
        "mov.b64 h0, {%2, %5};\n"
        "mov.b64 h1, {k1, %5};\n"
        "mov.b64 h2, {k2, %5};\n"
        "mov.b64 h3, {k3, %5};\n"
        "mov.b64 w0, {m0, %5};\n"
        "mov.b64 w1, {m1, %5};\n"
        "mov.b64 w2, {m2, %5};\n"
        "mov.b64 w3, {m3, %5};\n"
        "mov.b64 bb, {%3, %6};\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l0], h0, %4, {%7, %7, %7, %7}, pf;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], w0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l1], h1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], w1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l2], h2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], w2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l3], h3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], w3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ab], bb, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], h0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], h1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], h2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], h3, %4, {%7, %7, %7, %7}, pt;\n"
        "}\n" ::"r"(d),
        "r"(q), "r"(klo), "r"(blo), "r"(IDESC_QK64), "r"(kDescHiSw128), "r"(kDescHiBias), "r"(0u));
}
__device__ __forceinline__ void issue_score_half_lean_commit(uint32_t d, uint32_t q, uint32_t klo,
                                                      uint32_t blo, uint32_t bar) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b32 a1, a2, a3, l0, l1, l2, l3, ab, k1, k2, k3, m0, m1, m2, m3;\n"
        ".reg .b64 h0, h1, h2, h3, w0, w1, w2, w3, bb;\n"
        "setp.ne.b32 pf, %7, %7;\n"
        "setp.eq.b32 pt, %7, %7;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u32 l0, %1, 32;\n"
        "add.u32 l1, %1, 40;\n"
        "add.u32 l2, %1, 48;\n"
        "add.u32 l3, %1, 56;\n"
        "add.u32 ab, %1, 64;\n"
        "add.u32 k1, %2, 2;\n"
        "add.u32 k2, %2, 4;\n"
        "add.u32 k3, %2, 6;\n"
        "add.u32 m0, %2, 1024;\n"
        "add.u32 m1, %2, 1026;\n"
        "add.u32 m2, %2, 1028;\n"
        "add.u32 m3, %2, 1030;\n"
        "mov.b64 h0, {%2, %5};\n"
        "mov.b64 h1, {k1, %5};\n"
        "mov.b64 h2, {k2, %5};\n"
        "mov.b64 h3, {k3, %5};\n"
        "mov.b64 w0, {m0, %5};\n"
        "mov.b64 w1, {m1, %5};\n"
        "mov.b64 w2, {m2, %5};\n"
        "mov.b64 w3, {m3, %5};\n"
        "mov.b64 bb, {%3, %6};\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l0], h0, %4, {%7, %7, %7, %7}, pf;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], w0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l1], h1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], w1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l2], h2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], w2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l3], h3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], w3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ab], bb, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], h0, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], h1, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], h2, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], h3, %4, {%7, %7, %7, %7}, pt;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"
        "}\n" ::"r"(d),
        "r"(q), "r"(klo), "r"(blo), "r"(IDESC_QK64), "r"(kDescHiSw128), "r"(kDescHiBias), "r"(0u), "r"(bar)
        : "memory");
}

template <bool ELECT = false>
__device__ __forceinline__ void issue_score_half_tq(uint32_t d_tmem, uint32_t q, uint32_t kst,
                                                    int h) {
    const uint32_t kh = kst + uint32_t(h) * kHalfK;
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk) {
        umma_ts<ELECT>(d_tmem, q + 32 + kk * 8, umma_desc(kh + kk * 32, 1024, 2), IDESC_QK64,
                       kk > 0 ? 1u : 0u);
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kh + CHUNK + kk * 32, 1024, 2), IDESC_QK64,
                       1u);
    }
    umma_ts<ELECT>(d_tmem, q + 64, umma_desc(kst + QTILE + uint32_t(h) * kHalfB, 256, 6),
                   IDESC_QK64, 1u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kh + kk * 32, 1024, 2), IDESC_QK64, 1u);
}
template <bool ELECT = false>
__device__ __forceinline__ void issue_screen_half_tq(uint32_t d_tmem, uint32_t q, uint32_t kst,
                                                     int h) {
    const uint32_t kh = kst + uint32_t(h) * kHalfK;
    umma_ts<ELECT>(d_tmem, q + 64, umma_desc(kst + QTILE + uint32_t(h) * kHalfB, 256, 6),
                   IDESC_QK64, 0u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kh + kk * 32, 1024, 2), IDESC_QK64, 1u);
}

template <bool ELECT = false>
__device__ __forceinline__ void issue_screen_tile_tq(uint32_t d_tmem, uint32_t q, uint32_t kst) {
    umma_ts<ELECT>(d_tmem, q + 64, umma_desc(kst + QTILE, 256, 6), IDESC_QK, 0u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ts<ELECT>(d_tmem, q + kk * 8, umma_desc(kst + kk * 32, 1024, 2), IDESC_QK, 1u);
}

// Screening approximation t~ = bias + hi x hi (5 MMAs): only the hi chunk and the
// bias chunk of the key stage are read.
template <bool ELECT = false>
__device__ __forceinline__ void issue_screen_tile(uint32_t d_tmem, uint32_t qa, uint32_t ones,
                                                  uint32_t kst) {
    umma_ss<ELECT>(d_tmem, umma_desc(ones, 256, 6), umma_desc(kst + QTILE, 256, 6), IDESC_QK, 0u);
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ss<ELECT>(d_tmem, umma_desc(qa + kk * 32, 1024, 2), umma_desc(kst + kk * 32, 1024, 2),
                IDESC_QK, 1u);
}

// One 64-wide feature chunk of a score tile for d > 64 (operands streamed chunk
// by chunk). Two accumulators keep the fp32 rounding at the scale of each part:
// d_big = sum of hi x hi slices, then the bias on the last chunk (the bias
// ~ g/eps carries |y|^2/eps and can dwarf the dot product at large d, so adding
// it last keeps the 4 C roundings of the dot product at the dot product's own
// magnitude); d_small = the 8 cross terms per chunk (2^-11 of the score),
// summed by the epilogue.
template <bool ELECT = false>
__device__ __forceinline__ void issue_score_chunk(uint32_t d_big, uint32_t d_small, uint32_t qa,
                                                  uint32_t ka, uint32_t ones, uint32_t bias,
                                                  bool first, bool last) {
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk) {
        umma_ss<ELECT>(d_small, umma_desc(qa + CHUNK + kk * 32, 1024, 2), umma_desc(ka + kk * 32, 1024, 2),
                IDESC_QK, (first && kk == 0) ? 0u : 1u);
        umma_ss<ELECT>(d_small, umma_desc(qa + kk * 32, 1024, 2), umma_desc(ka + CHUNK + kk * 32, 1024, 2),
                IDESC_QK, 1u);
    }
#pragma unroll
    for (int kk = 0; kk < DPAD / 16; ++kk)
        umma_ss<ELECT>(d_big, umma_desc(qa + kk * 32, 1024, 2), umma_desc(ka + kk * 32, 1024, 2),
                IDESC_QK, (first && kk == 0) ? 0u : 1u);
    if (last) umma_ss<ELECT>(d_big, umma_desc(ones, 256, 6), umma_desc(bias, 256, 6), IDESC_QK, 1u);
}

}  // namespace tc
}  // namespace fskb
