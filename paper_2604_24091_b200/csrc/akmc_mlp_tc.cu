// akmc_mlp_tc.cu -- fused gather -> encode -> barrier MLP (3 x tcgen05) -> Arrhenius rates, sm_100a.
//
// Persistent kernel (<= one CTA per SM, 256 threads); each CTA loops over tiles of 128 vacancies:
//   G  gather the 64-site window of every row: one warp per row (lanes = slots j and
//      j+32) from the bricked halo storage, and the OR of the layer-1 K-steps the tile needs;
//   X  encode: K1 = 400, K-major SWIZZLE_128B in smem.  Columns 0,1 = 1 (the bias K-step), then a
//      species-major one-hot X[m][16 + 64(s-1) + slot] = [sigma_slot == s] over the 6 non-Fe species
//      (exact in fp16; the Fe column is folded into the bias, A5).  A K-step of 16 columns is all zero
//      for the tile unless some row holds species s in that 16-slot group: such K-steps are skipped
//      (they add exact zeros), so a dilute alloy streams ~6-8 of the 24 one-hot chunks;
//   M1 layer 1 on tcgen05: D1 = X*W1'hi, D2 = X*W1'lo, b1' inside the GEMM as three fp16 pieces
//      (W1' = W1 - W1[slot,Fe], scaled by 2^s1 and split hi + lo*2^-11; every product is exact, FP32
//      accumulation in TMEM);
//   E1 h1 = ReLU(2^-s1 (D1 + 2^-11 D2)), rounded to FP32, split into fp16 hi + lo*2^11 -> A (SW128);
//   M2 layer 2 (256x256, "swarm gathering" GEMM): D1 = Ahi*W2hi, D2 = Ahi*W2lo + Alo*W2hi;
//   E2 h2 = ReLU(2^-s2 (D1 + 2^-11 D2) + b2) -> split -> A;
//   M3 layer 3 (256x8 padded to N = 16) with 4 K-groups of 64 in separate TMEM accumulators;
//   E3 E = max(0, b3 + 2^-s3 sum_g (Da_g + 2^-11 Db_g)) in FP64; Gamma = nu0 det_exp(-E/kT), masked;
//      the two warp halves take hops 0-3 and 4-7 of a row.
// The needed W1' chunks and the 16 W2 chunks stream through one 4-stage cp.async.bulk + mbarrier ring
// (16 KiB per chunk, in ascending K order) driven by a single control thread that also issues every
// tcgen05.mma.  The 3-pass fp16 split is FP32-equivalent ("matrix multiplication ... executed in
// FP32"); DESIGN.md sec. 6.
#include "akmc_mlp_tc.cuh"
#include <cuda_fp16.h>

namespace akmc {

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kAtomBytes = kTileM * 128;  // one SW128 K-atom (64 fp16 of K) of a 128-row tile: 16 KiB
constexpr uint32_t kLboB = (kHid / 8) * 128;   // ring chunk split (N = 256, K = 16): K-dir core-matrix stride
constexpr uint32_t kLboW3 = (kN3 / 8) * 128;   // W3 image (N = 16): K-dir core-matrix stride = 256 B
constexpr uint32_t kSboNoSw = 128;             // no-swizzle 8-row group stride
constexpr uint32_t kSboA = 1024;               // SW128 8-row group stride
constexpr int kWinStride = 68;                 // window bytes per row in smem (17 words: conflict-free)

// smem carve-up (offsets from a 1024-aligned base)
constexpr size_t kOffA = 0;                                   // A_hi [0,64K), A_lo [64K,128K); X overlays [0,112K)
constexpr size_t kOffB = kOffA + 2 * (size_t)kABytes;         // ring 4 x 16 KiB
constexpr size_t kOffW3 = kOffB + (size_t)kStages * kStageBytes;   // W3 image 16 KiB
constexpr size_t kOffWin = kOffW3 + 2 * (size_t)kW3SplitBytes;     // uint8 [128][68]
constexpr size_t kOffB2 = kOffWin + (size_t)kTileM * kWinStride;   // float [256]
constexpr size_t kOffG = kOffB2 + kHid * 4;                        // double [128][4]
constexpr size_t kOffSlot = kOffG + (size_t)kTileM * 4 * 8;        // int [128]
constexpr size_t kOffMask = kOffSlot + kTileM * 4;                 // uint8 [128]
constexpr size_t kOffKmask = kOffMask + kTileM;                    // uint32 (+pad)
constexpr size_t kOffList = kOffKmask + 8;                         // uint8 [32]: the tile's W1' chunk ids
constexpr size_t kOffBar = kOffList + 32;                          // 8-B aligned barriers
constexpr int kNumBars = 2 * kStages + 4;                          // full[4], empty[4], done1..3, w3
constexpr size_t kOffTmem = kOffBar + kNumBars * 8;
constexpr size_t kSmemUsed = kOffTmem + 16;
constexpr size_t kSmemTotal = kSmemUsed + 1024;                    // alignment slack
static_assert(kSmemTotal <= 232448, "shared memory budget");
static_assert(kOffBar % 8 == 0, "barrier alignment");

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

__device__ __forceinline__ uint64_t desc_a(uint32_t base, int kstep)   // SW128 A/X operand, K-step of 16
{
    return umma_desc(base + (uint32_t)(kstep >> 2) * kAtomBytes + (uint32_t)(kstep & 3) * 32u, 16, kSboA, 2);
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
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_half2(__half a, __half b)
{
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// byte offset of (row m, 8-column group kg) in a K-major SWIZZLE_128B tile of 128 rows
__device__ __forceinline__ uint32_t sw128_off(int m, int kg)
{
    return (uint32_t)(kg >> 3) * kAtomBytes + (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u +
           (uint32_t)(((kg & 7) ^ (m & 7)) << 4);
}

// split 8 FP32 values into fp16 hi and lo*2^11 and store them at (m, kg) of the A tile
__device__ __forceinline__ void store_split8(uint8_t* A_hi, uint8_t* A_lo, int m, int kg, const float (&h)[8],
                                             unsigned long long& ovf)
{
    __half hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float v = h[i];
        if (v > 60000.0f) { v = 60000.0f; ++ovf; }
        hi[i] = __float2half_rn(v);
        lo[i] = __float2half_rn((v - __half2float(hi[i])) * kLoScale);
    }
    const uint32_t off = sw128_off(m, kg);
    *reinterpret_cast<uint4*>(A_hi + off) =
        make_uint4(pack_half2(hi[0], hi[1]), pack_half2(hi[2], hi[3]), pack_half2(hi[4], hi[5]), pack_half2(hi[6], hi[7]));
    *reinterpret_cast<uint4*>(A_lo + off) =
        make_uint4(pack_half2(lo[0], lo[1]), pack_half2(lo[2], lo[3]), pack_half2(lo[4], lo[5]), pack_half2(lo[6], lo[7]));
}

__global__ void __launch_bounds__(kThreads, 1) mlp_tc_kernel(const __grid_constant__ MlpTcParams p)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int nrows = p.nrows_dev ? *p.nrows_dev : p.nrows_host;
    const int ntiles = (nrows + kTileM - 1) / kTileM;
    if ((int)blockIdx.x >= ntiles) return;         // uniform early exit: no barrier/TMEM touched

    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* A_hi = smem + kOffA;
    uint8_t* A_lo = smem + kOffA + kABytes;
    uint8_t* Xs = smem + kOffA;                    // layer-1 operand overlays A
    uint8_t* Bst = smem + kOffB;
    uint8_t* W3s = smem + kOffW3;
    uint8_t* win = smem + kOffWin;
    float* sb2 = reinterpret_cast<float*>(smem + kOffB2);
    double* sG = reinterpret_cast<double*>(smem + kOffG);        // [128][4] rates of hops 4..7
    int* sslot = reinterpret_cast<int*>(smem + kOffSlot);
    uint8_t* smask = smem + kOffMask;
    uint32_t* skmask = reinterpret_cast<uint32_t*>(smem + kOffKmask);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t bar_full0 = smem_u32(&bars[0]);
    const uint32_t bar_empty0 = smem_u32(&bars[kStages]);
    const uint32_t bar_done1 = smem_u32(&bars[2 * kStages + 0]);
    const uint32_t bar_done2 = smem_u32(&bars[2 * kStages + 1]);
    const uint32_t bar_done3 = smem_u32(&bars[2 * kStages + 2]);
    const uint32_t bar_w3 = smem_u32(&bars[2 * kStages + 3]);
    const bool ctrl = (warp == 1 && lane == 0);    // control thread: ring loads + every tcgen05.mma

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_full0 + 8 * s, 1);
            mbar_init(bar_empty0 + 8 * s, 1);
        }
        mbar_init(bar_done1, 1);
        mbar_init(bar_done2, 1);
        mbar_init(bar_done3, 1);
        mbar_init(bar_w3, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *skmask = 1u;                              // K-step 0 (bias) is always needed
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(tmem_slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = threadIdx.x; i < kHid; i += kThreads) sb2[i] = p.b2[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc256 = (1u << 4) | ((uint32_t)(kHid >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
    const uint32_t idesc16 = (1u << 4) | ((uint32_t)(kN3 >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);

    // ring (control thread only): position y in stage y % 4; chunks in ascending K order per tile
    int issued = 0, consumed = 0;                  // ring positions over this CTA's whole life
    int tile_base = 0, tile_n = 0, n1 = 0;         // current tile: first position, entries, W1' entries
    uint8_t* list = smem + kOffList;               // W1' chunk ids needed by the current tile
    auto chunk_id = [&](int e) { return e < n1 ? (int)list[e] : kChunksL1 + (e - n1); };
    auto issue_next = [&]() {
        if (issued >= tile_base + tile_n) return;
        const int y = issued++;
        const int s = y % kStages;
        if (y >= kStages) mbar_wait(bar_empty0 + 8 * s, ((y - kStages) / kStages) & 1);
        mbar_expect_tx(bar_full0 + 8 * s, kStageBytes);
        bulk_g2s(smem_u32(Bst + (size_t)s * kStageBytes),
                 reinterpret_cast<const uint8_t*>(p.Bimg) + (size_t)chunk_id(y - tile_base) * kStageBytes, kStageBytes,
                 bar_full0 + 8 * s);
    };
    auto chunk_ready = [&]() {
        const int y = consumed;
        mbar_wait(bar_full0 + 8 * (y % kStages), (y / kStages) & 1);
        tc_fence_after();
        return smem_u32(Bst + (size_t)(y % kStages) * kStageBytes);
    };
    auto chunk_done = [&]() {
        umma_commit(bar_empty0 + 8 * (consumed % kStages));
        ++consumed;
        issue_next();                              // keeps kStages-1 chunks in flight
    };
    if (ctrl) {
        mbar_expect_tx(bar_w3, 2 * kW3SplitBytes);
        bulk_g2s(smem_u32(W3s), p.W3img, 2 * kW3SplitBytes, bar_w3);
    }

    const long long tk0 = clock64();
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int tile0 = tile * kTileM;
        long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const bool timing = p.phase_cycles && threadIdx.x == 64;
        if (timing) tp[0] = clock64();

        // ---- G: gather, one warp per row (lane = window slots j and j+32), 16 rows per warp in two
        //      batches of 8 so that the dependent loads (row -> vacancy -> window) overlap across rows;
        //      one LDG instruction then touches the ~10 bricks (L2 lines) of one window, not 32 windows.
        //      Also collects which layer-1 K-steps the tile needs (species-major groups of 16 slots).
        {
            const int ox0 = p.G.off[lane][0], oy0 = p.G.off[lane][1], oz0 = p.G.off[lane][2];
            const int ox1 = p.G.off[lane + 32][0], oy1 = p.G.off[lane + 32][1], oz1 = p.G.off[lane + 32][2];
            uint32_t kbits = 0;
#pragma unroll
            for (int half8 = 0; half8 < 2; ++half8) {
                uint32_t b0[8], b1[8];
                int sl[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int r = warp + 8 * (8 * half8 + i);
                    const int g = tile0 + r;
                    b0[i] = 0; b1[i] = 0; sl[i] = -1;
                    if (g < nrows) {
                        if (p.windows) {
                            sl[i] = g;
                            b0[i] = __ldg(p.windows + (size_t)g * kWin + lane);
                            b1[i] = __ldg(p.windows + (size_t)g * kWin + lane + 32);
                        } else {
                            const int slot = p.rows ? __ldg(p.rows + g) : g;
                            const int4 v = p.vac[slot];
                            sl[i] = slot;
                            b0[i] = __ldg(p.species + site_of(p.F, v.x, v.y + ox0, v.z + oy0, v.w + oz0));
                            b1[i] = __ldg(p.species + site_of(p.F, v.x, v.y + ox1, v.z + oy1, v.w + oz1));
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int r = warp + 8 * (8 * half8 + i);
                    win[r * kWinStride + lane] = (uint8_t)b0[i];
                    win[r * kWinStride + lane + 32] = (uint8_t)b1[i];
                    if (b0[i] != kFe) kbits |= 1u << (1 + 4 * (b0[i] - 1) + (lane >> 4));
                    if (b1[i] != kFe) kbits |= 1u << (1 + 4 * (b1[i] - 1) + 2 + (lane >> 4));
                    const unsigned feas = __ballot_sync(0xffffffffu, lane < kHops && b0[i] != (uint32_t)kVac);
                    if (lane == 0) {
                        smask[r] = (uint8_t)(feas & 0xFFu);
                        sslot[r] = sl[i];
                    }
                }
            }
            kbits = __reduce_or_sync(0xffffffffu, kbits);
            if (lane == 0 && kbits) atomicOr(skmask, kbits);
        }
        __syncthreads();
        if (ctrl) {
            // the tile's chunk list: needed W1' K-steps in ascending order, then the 16 W2 chunks
            const uint32_t km = *skmask;
            *skmask = 1u;                          // next OR comes after several __syncthreads
            n1 = 0;
            for (int c = 0; c < kChunksL1; ++c)
                if ((km >> c) & 1u) list[n1++] = (uint8_t)c;
            tile_base = issued;
            tile_n = n1 + kChunksL2;
            for (int q = 0; q < kStages - 1; ++q) issue_next();    // overlap with the encode
        }
        if (timing) tp[1] = clock64();

        // ---- X: one-hot layer-1 operand (K = 400, SW128): columns 0,1 = 1 (bias pieces), then
        //      column 16 + (s-1)*64 + slot.  Thread (row m, half hx) owns the chunks of window slots
        //      [32hx, 32hx+32) in every species block (plus the bias chunks for hx = 0): zero-fill them,
        //      then write fp16 1.0 for its non-Fe slots -- no other thread writes those chunks.
        {
            const int m = 32 * (warp & 3) + lane;
            const int hx = warp >> 2;
            const uint32_t* wr = reinterpret_cast<const uint32_t*>(win + m * kWinStride) + 8 * hx;
            uint32_t w32[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) w32[q] = wr[q];
            if (hx == 0) {
                *reinterpret_cast<uint4*>(Xs + sw128_off(m, 0)) = make_uint4(0x3C003C00u, 0u, 0u, 0u);
                *reinterpret_cast<uint4*>(Xs + sw128_off(m, 1)) = make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int s = 0; s < kSpecies - 1; ++s)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<uint4*>(Xs + sw128_off(m, 2 + 8 * s + 4 * hx + q)) = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
                const int s = (int)((w32[jj >> 2] >> (8 * (jj & 3))) & 0xFFu);
                if (s != kFe) {
                    const int f = 16 + kWin * (s - 1) + 32 * hx + jj;
                    *reinterpret_cast<__half*>(Xs + sw128_off(m, f >> 3) + 2 * (f & 7)) = __ushort_as_half(0x3C00);
                }
            }
        }
        fence_async_smem();
        __syncthreads();
        if (timing) tp[2] = clock64();

        // ---- M1: layer 1 on tcgen05 over the needed K-steps (skipped K-steps are all-zero: exact)
        if (ctrl) {
            tc_fence_after();
            const uint32_t xb = smem_u32(Xs);
            for (int e = 0; e < n1; ++e) {
                const uint32_t bh = chunk_ready();
                const uint64_t da = desc_a(xb, list[e]);
                umma_f16(tmem + 0, da, umma_desc(bh, kLboB, kSboNoSw, 0), idesc256, e > 0 ? 1u : 0u);
                umma_f16(tmem + kHid, da, umma_desc(bh + kSplitBytes, kLboB, kSboNoSw, 0), idesc256, e > 0 ? 1u : 0u);
                chunk_done();
            }
            umma_commit(bar_done1);
        }
        __syncwarp();
        mbar_wait(bar_done1, it & 1);
        tc_fence_after();
        if (timing) tp[3] = clock64();

        // ---- E1: h1 = ReLU(2^-s1 (D1 + 2^-11 D2)) (b1' is inside the GEMM) -> split -> A
        const int q4 = warp & 3, half = warp >> 2;
        const int row = 32 * q4 + lane;
        const uint32_t tlane = tmem + ((uint32_t)(32 * q4) << 16);
        unsigned long long ovf = 0;
        {
            const float s1 = p.s1_unscale, inv_lo = 1.0f / kLoScale;
            for (int cb = 0; cb < 8; ++cb) {
                const int col = half * 128 + cb * 16;
                uint32_t d1[16], d2[16];
                tmem_ld16(tlane + (uint32_t)col, d1);
                tmem_ld16(tlane + (uint32_t)(kHid + col), d2);
                tmem_wait_ld();
#pragma unroll
                for (int g8 = 0; g8 < 2; ++g8) {
                    float h[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float v = __fmaf_rn(__uint_as_float(d2[8 * g8 + i]), inv_lo, __uint_as_float(d1[8 * g8 + i])) * s1;
                        h[i] = v > 0.0f ? v : 0.0f;
                    }
                    store_split8(A_hi, A_lo, row, (col >> 3) + g8, h, ovf);
                }
            }
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (timing) tp[4] = clock64();

        // ---- M2: layer 2 on tcgen05 (16 K-steps; W2 hi/lo from the ring)
        if (ctrl) {
            tc_fence_after();
            const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo);
            for (int c = 0; c < kChunksL2; ++c) {
                const uint32_t bh = chunk_ready();
                const uint64_t dah = desc_a(ah, c), dal = desc_a(al, c);
                const uint64_t dbh = umma_desc(bh, kLboB, kSboNoSw, 0);
                const uint64_t dbl = umma_desc(bh + kSplitBytes, kLboB, kSboNoSw, 0);
                umma_f16(tmem + 0, dah, dbh, idesc256, c > 0 ? 1u : 0u);
                umma_f16(tmem + kHid, dah, dbl, idesc256, c > 0 ? 1u : 0u);
                umma_f16(tmem + kHid, dal, dbh, idesc256, 1u);
                chunk_done();
            }
            umma_commit(bar_done2);
        }
        __syncwarp();
        mbar_wait(bar_done2, it & 1);
        tc_fence_after();
        if (timing) tp[5] = clock64();

        // ---- E2: h2 = ReLU(2^-s2 (D1 + 2^-11 D2) + b2) -> split -> A
        {
            const float inv_lo = 1.0f / kLoScale;
            for (int cb = 0; cb < 8; ++cb) {
                const int col = half * 128 + cb * 16;
                uint32_t d1[16], d2[16];
                tmem_ld16(tlane + (uint32_t)col, d1);
                tmem_ld16(tlane + (uint32_t)(kHid + col), d2);
                tmem_wait_ld();
#pragma unroll
                for (int g8 = 0; g8 < 2; ++g8) {
                    float h[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int n = col + 8 * g8 + i;
                        float z = __fmaf_rn(__uint_as_float(d2[8 * g8 + i]), inv_lo, __uint_as_float(d1[8 * g8 + i]));
                        z = __fmaf_rn(z, p.s2_unscale, sb2[n]);
                        h[i] = z > 0.0f ? z : 0.0f;
                    }
                    store_split8(A_hi, A_lo, row, (col >> 3) + g8, h, ovf);
                }
            }
        }
        if (ovf && p.overflow) atomicAdd(p.overflow, ovf);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (timing) tp[6] = clock64();

        // ---- M3: layer 3 (N = 16), 4 K-groups x {hi*hi, hi*lo + lo*hi} accumulators in TMEM cols [0,128)
        if (ctrl) {
            if (it == 0) mbar_wait(bar_w3, 0);
            tc_fence_after();
            const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo), w3 = smem_u32(W3s);
            for (int c = 0; c < kHid / 16; ++c) {
                const uint32_t g = (uint32_t)(c >> 2);
                const uint32_t acc = (c & 3) ? 1u : 0u;
                const uint64_t dah = desc_a(ah, c), dal = desc_a(al, c);
                const uint64_t dbh = umma_desc(w3 + (uint32_t)c * 2 * kLboW3, kLboW3, kSboNoSw, 0);
                const uint64_t dbl = umma_desc(w3 + kW3SplitBytes + (uint32_t)c * 2 * kLboW3, kLboW3, kSboNoSw, 0);
                umma_f16(tmem + 32 * g, dah, dbh, idesc16, acc);
                umma_f16(tmem + 32 * g + 16, dah, dbl, idesc16, acc);
                umma_f16(tmem + 32 * g + 16, dal, dbh, idesc16, 1u);
            }
            umma_commit(bar_done3);
        }
        __syncwarp();
        mbar_wait(bar_done3, it & 1);
        tc_fence_after();

        // ---- E3: barriers and rates; warp half h handles hops [4h, 4h+4) of its row
        {
            double accE[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t da[8], db[8];
                tmem_ld8(tlane + (uint32_t)(32 * g), da);
                tmem_ld8(tlane + (uint32_t)(32 * g + 16), db);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    accE[k] += (double)__uint_as_float(da[4 * half + k]) +
                               (double)__uint_as_float(db[4 * half + k]) * (1.0 / 2048.0);
            }
            const int slot = sslot[row];
            double Gk[4];
            if (slot >= 0) {
                const int mask = smask[row];
                const double ikT = p.windows ? p.P.inv_kT : 1.0 / kT_of(p.P, max(p.vac[slot].x, 0));
                double Ek[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int kk = 4 * half + k;
                    const double out = __ldg(p.b3 + kk) + accE[k] * p.s3_unscale;
                    Ek[k] = out > 0.0 ? out : 0.0;
                    Gk[k] = ((mask >> kk) & 1) ? p.P.nu0 * det_exp(-(Ek[k] * ikT)) : 0.0;
                }
                if (p.E) {
                    double2* e2 = reinterpret_cast<double2*>(p.E + (size_t)slot * 8 + 4 * half);
                    e2[0] = make_double2(Ek[0], Ek[1]);
                    e2[1] = make_double2(Ek[2], Ek[3]);
                }
                if (p.rates) {
                    double2* g2 = reinterpret_cast<double2*>(p.rates + (size_t)slot * 8 + 4 * half);
                    g2[0] = make_double2(Gk[0], Gk[1]);
                    g2[1] = make_double2(Gk[2], Gk[3]);
                }
                if (half == 1) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) sG[row * 4 + k] = Gk[k];
                }
            }
            tc_fence_before();
            __syncthreads();
            if (half == 0 && slot >= 0 && p.Rsum) {
                double Rs = 0.0;                   // R = ((G0 + G1) + ...) + G7, fixed order
#pragma unroll
                for (int k = 0; k < 4; ++k) Rs = __dadd_rn(Rs, Gk[k]);
#pragma unroll
                for (int k = 0; k < 4; ++k) Rs = __dadd_rn(Rs, sG[row * 4 + k]);
                p.Rsum[slot] = Rs;
            }
        }
        __syncthreads();          // TMEM, A/X, window and sG buffers free for the next tile
        if (timing) {
            tp[7] = clock64();
            for (int ph = 0; ph < 7; ++ph) atomicAdd(p.phase_cycles + ph, (unsigned long long)(tp[ph + 1] - tp[ph]));
            atomicAdd(p.phase_cycles + 7, 1ull);
        }
    }
    if (p.phase_cycles && threadIdx.x == 64) {
        atomicAdd(p.phase_cycles + 8, (unsigned long long)(clock64() - tk0));   // CTA loop time
        atomicAdd(p.phase_cycles + 9, 1ull);                                    // CTAs with work
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
