// akmc_mlp_tc.cu -- fused gather -> encode -> barrier MLP (tcgen05) -> Arrhenius rates, sm_100a.
//
// Persistent kernel (<= one CTA per SM); each CTA loops over tiles of 128 vacancies (rows):
//   1. gather the 64-site window of every row and encode it sparsely: the
//      one-hot 448-vector is summarised by its non-Fe features f = 7*slot + species (A5);
//   2. layer 1 as a Fe-referenced embedding bag accumulated in FP64 (exact algebra: the Fe rows
//      are folded into the bias); one warp per row, lanes over columns, coalesced 2 KiB W1' rows;
//      ReLU, rounded to FP32 and split into fp16 hi + lo*2^11, stored K-major SWIZZLE_128B;
//   3. layer 2 (256x256, "swarm gathering" GEMM) on the 5th-gen tensor cores:
//      D1 = Ahi*Bhi, D2 = Ahi*Blo + Alo*Bhi accumulated in TMEM (FP32); W2 streamed through a
//      4-stage cp.async.bulk + mbarrier ring; one elected thread issues tcgen05.mma;
//   4. epilogue from TMEM (tcgen05.ld): h2 = ReLU(D1 + 2^-11 D2 + b2), layer 3 (256x8) as FP32
//      16-term partials folded into FP64, E = max(0, out), Gamma = nu0 * det_exp(-E/kT) with the
//      feasibility mask (Eq. 1, Eq. 8).
// The split is FP32-equivalent (22-bit products, FP32 accumulation), the paper's "matrix
// multiplication ... executed in FP32"; DESIGN.md sec. 6 gives the error budget.
#include "akmc_mlp_tc.cuh"
#include <cuda_fp16.h>

namespace akmc {

namespace {

constexpr int kThreads = 256;
constexpr int kNnzCap = kWin;                  // non-Fe features per row (<= 64)
constexpr uint32_t kAtomBytes = kTileM * 128;  // one SW128 K-atom (64 fp16 of K) of the A tile: 16 KiB
constexpr uint32_t kLboB = (kHid / 8) * 128;   // K-direction core-matrix stride of a B chunk split: 4096 B
constexpr uint32_t kSboB = 128;                // B: 8-row group stride (no swizzle)
constexpr uint32_t kSboA = 1024;               // A: 8-row group stride (SWIZZLE_128B atom)

// smem carve-up (offsets from a 1024-aligned base)
constexpr size_t kOffAhi = 0;
constexpr size_t kOffAlo = kOffAhi + kABytes;
constexpr size_t kOffB = kOffAlo + kABytes;
constexpr size_t kOffNnz = kOffB + (size_t)kStages * kStageBytes;      // uint16 [128][64] (reused: double [128][8])
constexpr size_t kOffW3 = kOffNnz + (size_t)kTileM * kNnzCap * 2;      // float [256][8]
constexpr size_t kOffB2 = kOffW3 + (size_t)kHid * 8 * 4;               // float [256]
constexpr size_t kOffB1 = kOffB2 + (size_t)kHid * 4;                   // double [256]
constexpr size_t kOffSlot = kOffB1 + (size_t)kHid * 8;                 // int [128]
constexpr size_t kOffCnt = kOffSlot + (size_t)kTileM * 4;              // uint8 [128]
constexpr size_t kOffMask = kOffCnt + kTileM;                          // uint8 [128]
constexpr size_t kOffBar = kOffMask + kTileM;                          // 8-B aligned
constexpr size_t kOffTmem = kOffBar + 16 * 8;
constexpr size_t kSmemUsed = kOffTmem + 16;
constexpr size_t kSmemTotal = kSmemUsed + 1024;                        // alignment slack
static_assert(kSmemTotal <= 232448, "shared memory budget");

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// UMMA shared-memory descriptors, K-major.  layout: 0 = SWIZZLE_NONE, 2 = SWIZZLE_128B (bits 61-63)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_half2(__half a, __half b)
{
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// byte offset of (row m, 8-column group kg) in a K-major SWIZZLE_128B A tile of 128 rows x 256 K
__device__ __forceinline__ uint32_t a_sw128_off(int m, int kg)
{
    return (uint32_t)(kg >> 3) * kAtomBytes + (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u +
           (uint32_t)(((kg & 7) ^ (m & 7)) << 4);
}

__global__ void __launch_bounds__(kThreads, 1) mlp_tc_kernel(const __grid_constant__ MlpTcParams p)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int nrows = p.nrows_dev ? *p.nrows_dev : p.nrows_host;
    const int ntiles = (nrows + kTileM - 1) / kTileM;
    if ((int)blockIdx.x >= ntiles) return;         // uniform early exit: no barrier/TMEM touched

    // 1024-B aligned base, keeping shared-space provenance (so accesses compile to LDS/STS)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* A_hi = smem + kOffAhi;
    uint8_t* A_lo = smem + kOffAlo;
    uint8_t* Bst = smem + kOffB;
    uint16_t* nnz = reinterpret_cast<uint16_t*>(smem + kOffNnz);
    float* sW3 = reinterpret_cast<float*>(smem + kOffW3);
    float* sb2 = reinterpret_cast<float*>(smem + kOffB2);
    double* sb1 = reinterpret_cast<double*>(smem + kOffB1);
    int* sslot = reinterpret_cast<int*>(smem + kOffSlot);
    uint8_t* scnt = smem + kOffCnt;
    uint8_t* smask = smem + kOffMask;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);   // full[4], empty[4], done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
    double* spartd = reinterpret_cast<double*>(smem + kOffNnz);    // aliases nnz after layer 1

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t bar_full0 = smem_u32(&bars[0]);
    const uint32_t bar_empty0 = smem_u32(&bars[kStages]);
    const uint32_t bar_done = smem_u32(&bars[2 * kStages]);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_full0 + 8 * s, 1);
            mbar_init(bar_empty0 + 8 * s, 1);
        }
        mbar_init(bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < kHid * 8; i += kThreads) sW3[i] = p.W3[i];
    for (int i = threadIdx.x; i < kHid; i += kThreads) { sb2[i] = p.b2[i]; sb1[i] = p.b1p[i]; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = (1u << 4)                         // D = F32
                         | ((uint32_t)(kHid >> 3) << 17)     // N = 256
                         | ((uint32_t)(kTileM >> 4) << 24);  // M = 128; A, B = F16, K-major

    // W2 chunk gc (global over this CTA's tiles) lives in stage gc % kStages; its u-th use is u = gc / kStages
    auto load_chunk = [&](int gc) {
        const int s = gc % kStages;
        const int u = gc / kStages;
        if (u > 0) mbar_wait(bar_empty0 + 8 * s, (u - 1) & 1);
        mbar_expect_tx(bar_full0 + 8 * s, kStageBytes);
        bulk_g2s(smem_u32(Bst + (size_t)s * kStageBytes),
                 reinterpret_cast<const uint8_t*>(p.Bimg) + (size_t)(gc % kNChunks) * kStageBytes, kStageBytes,
                 bar_full0 + 8 * s);
    };

    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int tile0 = tile * kTileM;
        const int gc0 = it * kNChunks;
        // producer: the first stages of W2 stream in while the rows are gathered and encoded
        if (threadIdx.x == 0)
            for (int c = 0; c < kStages; ++c) load_chunk(gc0 + c);

        // ---- gather + sparse encode (threads 0..127, one row each)
        if (threadIdx.x < kTileM) {
            const int r = threadIdx.x;
            const int g = tile0 + r;
            int cnt = 0, mask = 0, slot = -1;
            if (g < nrows) {
                uint8_t w[kWin];
                if (p.windows) {
                    slot = g;
                    const uint4* src = reinterpret_cast<const uint4*>(p.windows + (size_t)g * kWin);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 v = __ldg(src + q);
                        const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int b = 0; b < 16; ++b) w[16 * q + b] = (uint8_t)(wd[b >> 2] >> (8 * (b & 3)));
                    }
                } else {
                    slot = p.rows ? p.rows[g] : g;
                    const int4 v = p.vac[slot];
#pragma unroll
                    for (int j = 0; j < kWin; ++j)
                        w[j] = __ldg(p.species + neighbour_site(p.F, v, p.G.off[j][0], p.G.off[j][1], p.G.off[j][2]));
                }
#pragma unroll
                for (int j = 0; j < kWin; ++j) {
                    const int s = w[j];
                    if (s != kFe) nnz[r * kNnzCap + (cnt++)] = (uint16_t)(kSpecies * j + s);
                    if (j < kHops && s != kVac) mask |= 1 << j;
                }
            }
            scnt[r] = (uint8_t)cnt;
            smask[r] = (uint8_t)mask;
            sslot[r] = slot;
        }
        __syncthreads();

        // ---- layer 1: one warp per row (4 rows in flight), lane = 8-column group; FP64 accumulate
        {
            double bias[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) bias[i] = sb1[lane * 8 + i];
            unsigned long long ovf = 0;
            for (int grp = 0; grp < kTileM / 32; ++grp) {
                int rr[4], cc[4];
                int nmax = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    rr[j] = warp + 8 * (4 * grp + j);
                    cc[j] = scnt[rr[j]];
                    nmax = max(nmax, cc[j]);
                }
                double acc[4][8];
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[j][i] = bias[i];
                for (int q = 0; q < nmax; ++q) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (q < cc[j]) {
                            const int f = nnz[rr[j] * kNnzCap + q];
                            const double2* wp = reinterpret_cast<const double2*>(p.W1p + (size_t)f * kHid + lane * 8);
                            const double2 x0 = __ldg(wp), x1 = __ldg(wp + 1), x2 = __ldg(wp + 2), x3 = __ldg(wp + 3);
                            acc[j][0] += x0.x; acc[j][1] += x0.y; acc[j][2] += x1.x; acc[j][3] += x1.y;
                            acc[j][4] += x2.x; acc[j][5] += x2.y; acc[j][6] += x3.x; acc[j][7] += x3.y;
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    __half hi[8], lo[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float h = (float)(acc[j][i] > 0.0 ? acc[j][i] : 0.0);
                        if (h > 60000.0f) { h = 60000.0f; ++ovf; }
                        hi[i] = __float2half_rn(h);
                        lo[i] = __float2half_rn((h - __half2float(hi[i])) * kLoScale);
                    }
                    const uint32_t off = a_sw128_off(rr[j], lane);
                    *reinterpret_cast<uint4*>(A_hi + off) = make_uint4(pack_half2(hi[0], hi[1]), pack_half2(hi[2], hi[3]),
                                                                       pack_half2(hi[4], hi[5]), pack_half2(hi[6], hi[7]));
                    *reinterpret_cast<uint4*>(A_lo + off) = make_uint4(pack_half2(lo[0], lo[1]), pack_half2(lo[2], lo[3]),
                                                                       pack_half2(lo[4], lo[5]), pack_half2(lo[6], lo[7]));
                }
            }
            if (ovf && p.overflow) atomicAdd(p.overflow, ovf);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
        __syncthreads();

        // ---- roles: W2 producer (warp 0), MMA issuer (warp 1)
        if (warp == 0) {
            if (lane == 0)
                for (int c = kStages; c < kNChunks; ++c) load_chunk(gc0 + c);
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0) {
                tc_fence_after();
                const uint32_t a_hi = smem_u32(A_hi), a_lo = smem_u32(A_lo);
                for (int c = 0; c < kNChunks; ++c) {        // one UMMA K-step (16) per chunk
                    const int gc = gc0 + c;
                    const int s = gc % kStages;
                    mbar_wait(bar_full0 + 8 * s, (gc / kStages) & 1);
                    tc_fence_after();
                    const uint32_t aoff = (uint32_t)(c >> 2) * kAtomBytes + (uint32_t)(c & 3) * 32u;
                    const uint64_t dah = umma_desc(a_hi + aoff, 16, kSboA, 2);
                    const uint64_t dal = umma_desc(a_lo + aoff, 16, kSboA, 2);
                    const uint32_t b_hi = smem_u32(Bst + (size_t)s * kStageBytes);
                    const uint64_t dbh = umma_desc(b_hi, kLboB, kSboB, 0);
                    const uint64_t dbl = umma_desc(b_hi + kSplitBytes, kLboB, kSboB, 0);
                    umma_f16(tmem + 0, dah, dbh, idesc, c > 0 ? 1u : 0u);
                    umma_f16(tmem + kHid, dah, dbl, idesc, c > 0 ? 1u : 0u);
                    umma_f16(tmem + kHid, dal, dbh, idesc, 1u);
                    umma_commit(bar_empty0 + 8 * s);       // stage free once these MMAs retire
                }
                umma_commit(bar_done);
            }
            __syncwarp();
        }

        // ---- epilogue: TMEM -> registers, ReLU, layer 3, rates
        mbar_wait(bar_done, it & 1);
        tc_fence_after();
        {
            const int q = warp & 3;
            const int half = warp >> 2;
            const int row = 32 * q + lane;
            const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16);
            // layer 3: FP32 products summed in chunks of 16 columns, chunk partials folded into FP64
            // (a single long FP32 chain loses ~1e-6 eV when one large gate term dominates the sum)
            double acc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = 0.0;
            const float inv_lo = 1.0f / kLoScale;
            for (int cb = 0; cb < 8; ++cb) {
                const int col = half * 128 + cb * 16;
                uint32_t d1[16], d2[16];
                tmem_ld16(tbase + (uint32_t)col, d1);
                tmem_ld16(tbase + (uint32_t)(kHid + col), d2);
                tmem_wait_ld();
                float part[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) part[k] = 0.0f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int n = col + i;
                    float z = fmaf(__uint_as_float(d2[i]), inv_lo, __uint_as_float(d1[i]));
                    z = fmaf(z, p.w2_unscale, sb2[n]);
                    const float h = fmaxf(z, 0.0f);
                    const float4 w0 = *reinterpret_cast<const float4*>(sW3 + n * 8);
                    const float4 w1 = *reinterpret_cast<const float4*>(sW3 + n * 8 + 4);
                    part[0] = fmaf(h, w0.x, part[0]); part[1] = fmaf(h, w0.y, part[1]);
                    part[2] = fmaf(h, w0.z, part[2]); part[3] = fmaf(h, w0.w, part[3]);
                    part[4] = fmaf(h, w1.x, part[4]); part[5] = fmaf(h, w1.y, part[5]);
                    part[6] = fmaf(h, w1.z, part[6]); part[7] = fmaf(h, w1.w, part[7]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] += (double)part[k];
            }
            if (half == 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k) spartd[row * 8 + k] = acc[k];
            }
            tc_fence_before();
            __syncthreads();
            if (half == 0) {
                const int slot = sslot[row];
                if (slot >= 0) {
                    const int mask = smask[row];
                    double Rs = 0.0;
                    double Ek[8], Gk[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const double out = (acc[k] + spartd[row * 8 + k]) + (double)__ldg(p.b3 + k);
                        Ek[k] = out > 0.0 ? out : 0.0;
                        Gk[k] = ((mask >> k) & 1) ? arrhenius(Ek[k], p.P) : 0.0;
                        Rs = __dadd_rn(Rs, Gk[k]);
                    }
                    if (p.E) {
                        double2* e2 = reinterpret_cast<double2*>(p.E + (size_t)slot * 8);
#pragma unroll
                        for (int k = 0; k < 4; ++k) e2[k] = make_double2(Ek[2 * k], Ek[2 * k + 1]);
                    }
                    if (p.rates) {
                        double2* g2 = reinterpret_cast<double2*>(p.rates + (size_t)slot * 8);
#pragma unroll
                        for (int k = 0; k < 4; ++k) g2[k] = make_double2(Gk[2 * k], Gk[2 * k + 1]);
                    }
                    if (p.Rsum) p.Rsum[slot] = Rs;
                }
            }
        }
        __syncthreads();          // spart/nnz and TMEM free for the next tile
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

} // namespace

size_t mlp_tc_smem_bytes() { return kSmemTotal; }

cudaError_t mlp_tc_setup()
{
    return cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTotal);
}

cudaError_t launch_mlp_tc(const MlpTcParams& p, int max_rows, int num_sms, cudaStream_t s)
{
    if (max_rows <= 0) return cudaSuccess;
    int grid = (max_rows + kTileM - 1) / kTileM;      // persistent: at most one CTA per SM
    if (grid > num_sms) grid = num_sms;
    mlp_tc_kernel<<<grid, kThreads, kSmemTotal, s>>>(p);
    return cudaGetLastError();
}

} // namespace akmc
