// akmc_eval.cuh -- device pieces of the FP32-equivalent barrier-network evaluation shared by the phase engine
// (akmc_engine.cu) and the bulk evaluator (akmc_bulk.cu).  Both evaluate a window with exactly this arithmetic,
// so a row's result is one function of its window whichever kernel computes it (R7 row purity):
//   layer 1  h1 = ReLU(b1' + sum of the W1' rows of the window's non-Fe slots), FP64 sum in slot order, one
//            rounding to FP32, scaled by 2^-t1, split fp16 hi + lo * 2^11 (layer1_rows / l1_store);
//   layer 2  D1 = A_hi W2_hi, D2 = A_hi W2_lo + A_lo W2_hi on tcgen05 (kind::f16, FP32 accumulate), K-steps of
//            16 in ascending order, D2's two products per K-step in that order (issued by each kernel);
//   E2       h2_c = max(0, fma(fma(D2_c, 2^-11, D1_c), s2u, b2_c)) in FP32 (e2_chunk);
//   layer 3  FP64 on CUDA cores, chunk sums P_q and their fixed tree (l3_chunk; see the comment there);
//   E3       E_k = max(0, b3_k + acc_k), Gamma_k = nu0 det_exp(-E_k * (1/kT)) unless hop k is masked, R in hop order.
#pragma once
#include "akmc_engine.cuh"
#include "akmc_ptx.cuh"

#ifndef AKMC_L1_ROWS
#define AKMC_L1_ROWS 2          // layer-1 rows per warp in flight (4: register spills, slower)
#endif
#ifndef AKMC_L1_BATCH
#define AKMC_L1_BATCH 2         // W1' rows per layer-1 row in flight
#endif
#ifndef AKMC_W1_EVICT_LAST
#define AKMC_W1_EVICT_LAST 0    // L2 evict_last policy on W1' loads (no effect measured)
#endif

namespace akmc {
namespace {
using namespace ptx;

constexpr uint32_t kRowGroupA = (kHid / 8) * 128;              // 4096 B: one 8-row group of h1 (K-major no-swizzle)
constexpr float kLo = 2048.0f;                                 // fp16 lo parts carry the remainder * 2^11
constexpr int kL1List = 4;                                     // W1' row indices kept per row (RPV: ~1.6; more -> window path)

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// fp16 hi/lo split of an FP32 value (lo carries the remainder * 2^11)
// (the init-time activation scales keep v <= 2^15; a value beyond 60000 would be a bound violation: it is
// clamped, counted, and the call that produced it returns AKMC_ERR_RUNTIME)
__device__ __forceinline__ void split_h(float v, __half& hi, __half& lo, unsigned long long& ovf, bool count = true)
{
    if (v > 60000.0f) { v = 60000.0f; if (count) ++ovf; }
    hi = __float2half_rn(v);
    lo = __float2half_rn((v - __half2float(hi)) * kLo);
}

__device__ __forceinline__ uint4 pack8(const __half (&x)[8])
{
    return make_uint4(pack_half2(x[0], x[1]), pack_half2(x[2], x[3]), pack_half2(x[4], x[5]), pack_half2(x[6], x[7]));
}

// Layer 3 (h2 -> 8 barriers) on CUDA cores in FP64, the contract shared with the bulk evaluator
// (akmc_bulk.cu): h2 columns are taken in chunks of 16 (chunk q = global columns 16q..16q+15);
// P_q[k] = sequential fma over the chunk's 16 columns of (double)h2_c * W3[c][k] from 0;
// S_r = (P_{4r} + P_{4r+1}) + (P_{4r+2} + P_{4r+3}); out_k = b3_k + (((0 + S_0) + S_1) + S_2) + S_3.
// h2_c is the FP32 value max(0, fma(fma(D2, 2^-11, D1), s2u, b2_c)) -- products and sums in FP64, so layer 3
// adds no rounding beyond FP64 (it used to be a 3-pass fp16 tcgen05 product with FP32 accumulators).
__device__ __forceinline__ void l3_chunk(const float (&z)[16], const double* __restrict__ w3, double (&P)[8])
{
#pragma unroll
    for (int k = 0; k < 8; ++k) P[k] = 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        const double zt = (double)z[t];
#pragma unroll
        for (int k = 0; k < 8; ++k) P[k] = __fma_rn(zt, w3[t * 8 + k], P[k]);
    }
}

// h2 of 16 columns from the layer-2 accumulators (FP32-equivalent: D1 + 2^-11 D2), the E2 arithmetic
__device__ __forceinline__ void e2_chunk(const uint32_t (&d1)[16], const uint32_t (&d2)[16], const float* __restrict__ b2,
                                         float s2u, float (&z)[16])
{
    const float inv = 1.0f / kLo;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        float v = __fmaf_rn(__uint_as_float(d2[t]), inv, __uint_as_float(d1[t]));
        v = __fmaf_rn(v, s2u, b2[t]);
        z[t] = v > 0.0f ? v : 0.0f;
    }
}


// window byte of an owned vacancy (plain coherent load -- the lattice is written by this kernel), with the
// offset packed into a register (bytes dx, dy, dz): a lane-dependent index into the kernel
// parameters would be a divergent constant-cache load (serialised over the 32 addresses)
__device__ __forceinline__ uint32_t pack_off(const int8_t* o)
{
    return (uint32_t)(uint8_t)o[0] | ((uint32_t)(uint8_t)o[1] << 8) | ((uint32_t)(uint8_t)o[2] << 16);
}
__device__ __forceinline__ uint8_t site_byte_pk(const uint8_t* species, const Frame& F, const int4& v, uint32_t pk)
{
    return species[neighbour_site(F, v, (int)(int8_t)(pk & 0xFFu), (int)(int8_t)((pk >> 8) & 0xFFu),
                                  (int)(int8_t)((pk >> 16) & 0xFFu))];
}


// non-Fe slots of a window as two ballot masks (slots 0-31, 32-63); entry e of the slot-ordered list is the
// e-th set bit (no list is stored: the masks are warp-uniform registers)
struct L1Masks { unsigned m0, m1; int c0, n; };
constexpr int kL1Batch = AKMC_L1_BATCH;                  // W1' rows per row in flight (an RPV window has ~1.6 non-Fe slots)
__device__ __forceinline__ L1Masks l1_masks(const uint8_t* w)
{
    const int lane = threadIdx.x & 31;
    L1Masks r;
    r.m0 = __ballot_sync(0xffffffffu, w[lane] != (uint8_t)kFe);
    r.m1 = __ballot_sync(0xffffffffu, w[lane + 32] != (uint8_t)kFe);
    r.c0 = __popc(r.m0);
    r.n = r.c0 + __popc(r.m1);
    return r;
}
__device__ __forceinline__ int l1_row_index(const uint8_t* w, const L1Masks& k, int e)
{
    const int slot = e < k.c0 ? (int)__fns(k.m0, 0, e + 1) : 32 + (int)__fns(k.m1, 0, e - k.c0 + 1);
    return 1 + ((int)w[slot] - 1) * kWin + slot;
}

// the gather's by-product for layer 1: the row's non-Fe slots as W1' row indices, in slot order, from the
// window bytes held by the lanes (lane = slots lane, lane + 32); rows with more than kL1List fall back to the
// window in the global scratch
__device__ __forceinline__ void l1_list_store(int r, uint8_t b0, uint8_t b1, uint8_t* l1n, uint16_t* l1l)
{
    const int lane = threadIdx.x & 31;
    const unsigned m0 = __ballot_sync(0xffffffffu, b0 != (uint8_t)kFe);
    const unsigned m1 = __ballot_sync(0xffffffffu, b1 != (uint8_t)kFe);
    const unsigned lt = lanemask_lt();
    const int c0 = __popc(m0);
    if (lane == 0) l1n[r] = (uint8_t)(c0 + __popc(m1));
    if (b0 != (uint8_t)kFe) {
        const int e = __popc(m0 & lt);
        if (e < kL1List) l1l[r * kL1List + e] = (uint16_t)(1 + ((int)b0 - 1) * kWin + lane);
    }
    if (b1 != (uint8_t)kFe) {
        const int e = c0 + __popc(m1 & lt);
        if (e < kL1List) l1l[r * kL1List + e] = (uint16_t)(1 + ((int)b1 - 1) * kWin + lane + 32);
    }
}

__device__ __forceinline__ void l1_store(const double (&acc)[8], int m, uint8_t* A_hi, uint8_t* A_lo, uint8_t* g_hi,
                                         uint8_t* g_lo, unsigned long long& ovf, bool fast, float sc)
{
    const int lane = threadIdx.x & 31;
    __half hi[8], lo[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float h = (float)acc[c];
        h = h > 0.0f ? h : 0.0f;
        split_h(h * sc, hi[c], lo[c], ovf);          // sc = 2^-t1 (exact; 1 for O(1) activations)
    }
    const uint32_t off = (uint32_t)(m >> 3) * kRowGroupA + (uint32_t)lane * 128u + (uint32_t)(m & 7) * 16u;
    const uint4 vh = pack8(hi), vl = pack8(lo);
    *reinterpret_cast<uint4*>(A_hi + off) = vh;
    if (!fast) *reinterpret_cast<uint4*>(A_lo + off) = vl;
    // the same 16 B into the L2 staging block of this CTA (row m % kRoundRows of its block)
    const uint32_t goff = (uint32_t)((m % kRoundRows) >> 3) * kRowGroupA + (uint32_t)lane * 128u + (uint32_t)(m & 7) * 16u;
#if !AKMC_XCHG_DSMEM
    if (g_hi) {                                      // (the bulk evaluator has no staging copy)
        *reinterpret_cast<uint4*>(g_hi + goff) = vh;
        if (!fast) *reinterpret_cast<uint4*>(g_lo + goff) = vl;
    }
#endif
}

// layer 1 of up to kL1Rows rows (one warp), all loads of a batch in flight at once; b1s = a shared-memory copy
// of b1' (row 0 of W1'), or nullptr to read it from W1f (same values, so the same bits)
// (R rows per call, B W1' rows per row per batch: a per-kernel register trade-off; the per-row sum order -- b1' then
// the listed rows in slot order -- is the same for every R and B, so are the bits)
constexpr int kL1Rows = AKMC_L1_ROWS;
template <int kR = kL1Rows, int kB = kL1Batch>
__device__ __forceinline__ void layer1_rows(const int (&rr)[kR], int nv, const uint8_t* win, const uint8_t* l1n,
                                            const uint16_t* l1l, const float* __restrict__ W1f,
                                            const int (&m)[kR], uint8_t* A_hi, uint8_t* A_lo,
                                            uint8_t* g_hi, uint8_t* g_lo, unsigned long long& ovf, bool fast,
                                            float sc, long long* lp = nullptr, const float* b1s = nullptr)
{
    constexpr int kL1Rows = kR, kL1Batch = kB;
    const int lane = threadIdx.x & 31;
    long long t0 = lp ? clock64() : 0;
    auto plap = [&](int i) { if (lp) { const long long t = clock64(); lp[i] += t - t0; t0 = t; } };
    int n[kL1Rows];
    L1Masks k[kL1Rows];
    int nmax = 0;
#pragma unroll
    for (int r = 0; r < kL1Rows; ++r) {
        n[r] = r < nv ? (int)l1n[rr[r]] : 0;
        nmax = n[r] > nmax ? n[r] : nmax;
        k[r].m0 = 0u; k[r].m1 = 0u; k[r].c0 = 0; k[r].n = n[r];
        if (n[r] > kL1List) k[r] = l1_masks(win + rr[r] * kWin);    // rare crowded window (warp-uniform)
    }
    plap(0);
    const float4* base = reinterpret_cast<const float4*>(W1f) + 2 * lane;
#if AKMC_W1_EVICT_LAST
    const uint64_t pol = policy_evict_last();
#endif
    double a[kL1Rows][8];
    {
        float4 x0, x1;
        if (b1s) {
            x0 = reinterpret_cast<const float4*>(b1s)[2 * lane];
            x1 = reinterpret_cast<const float4*>(b1s)[2 * lane + 1];
        } else {
            x0 = __ldg(base); x1 = __ldg(base + 1);
        }
#pragma unroll
        for (int r = 0; r < kL1Rows; ++r) {
            a[r][0] = x0.x; a[r][1] = x0.y; a[r][2] = x0.z; a[r][3] = x0.w;
            a[r][4] = x1.x; a[r][5] = x1.y; a[r][6] = x1.z; a[r][7] = x1.w;
        }
    }
    plap(1);
    for (int e = 0; e < nmax; e += kL1Batch) {
        float4 xa[kL1Rows][kL1Batch], xb[kL1Rows][kL1Batch];
#pragma unroll
        for (int t = 0; t < kL1Batch; ++t) {
#pragma unroll
            for (int r = 0; r < kL1Rows; ++r) {
                if (e + t < n[r]) {
                    const int ix = n[r] <= kL1List ? (int)l1l[rr[r] * kL1List + e + t]
                                                   : l1_row_index(win + rr[r] * kWin, k[r], e + t);
                    const float4* rp = base + (size_t)ix * (kHid / 4);
#if AKMC_W1_EVICT_LAST
                    xa[r][t] = ldg_f4_hint(rp, pol); xb[r][t] = ldg_f4_hint(rp + 1, pol);
#else
                    xa[r][t] = __ldg(rp); xb[r][t] = __ldg(rp + 1);
#endif
                }
            }
        }
#pragma unroll
        for (int t = 0; t < kL1Batch; ++t) {
#pragma unroll
            for (int r = 0; r < kL1Rows; ++r) {
                if (e + t < n[r]) {
                    a[r][0] = __dadd_rn(a[r][0], (double)xa[r][t].x); a[r][1] = __dadd_rn(a[r][1], (double)xa[r][t].y);
                    a[r][2] = __dadd_rn(a[r][2], (double)xa[r][t].z); a[r][3] = __dadd_rn(a[r][3], (double)xa[r][t].w);
                    a[r][4] = __dadd_rn(a[r][4], (double)xb[r][t].x); a[r][5] = __dadd_rn(a[r][5], (double)xb[r][t].y);
                    a[r][6] = __dadd_rn(a[r][6], (double)xb[r][t].z); a[r][7] = __dadd_rn(a[r][7], (double)xb[r][t].w);
                }
            }
        }
    }
    plap(2);
#pragma unroll
    for (int r = 0; r < kL1Rows; ++r)
        if (r < nv) l1_store(a[r], m[r], A_hi, A_lo, g_hi, g_lo, ovf, fast, sc);
    __syncwarp();
    plap(3);
}

} // namespace
} // namespace akmc
