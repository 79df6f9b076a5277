// akmc_bulk.cu -- the bulk barrier-network evaluator: every row of a large batch (all vacancies of a block for
// akmc_rates, caller windows for akmc_eval_windows, the grid-synchronous loop's active sets) through the
// 448-256-256-8 network (sec. V.B.1 "swarm gathering": batched weight-sharing GEMVs as one
// GEMM), FP32-equivalent, with exactly the per-row arithmetic of the phase engine's cluster evaluator
// (akmc_eval.cuh), so every path that forms a rate forms the same bits (R7).
//
// One persistent CTA per SM, 128-row tiles, warp-specialised so that the tensor pipe, the FP64 pipe and the
// memory system work at the same time:
//   warps 0-3   epilogue: TMEM lane quadrant w; E2 (h2 in FP32), layer 3 (FP64 FMAs), E3 (Arrhenius, R);
//   warp  4     W2 loader: cp.async.bulk of the fp16 hi|lo image of one K-step of W2 (16 KB) into a 4-stage ring;
//   warp  5     MMA issuer (one thread): 16 K-steps x {D1 += Ahi W2hi, D2 += Ahi W2lo, D2 += Alo W2hi}, M=128
//               N=256 K=16, accumulators D1 | D2 = all 512 TMEM columns;
//   warps 6-15  producers: gather the next tile's windows (while the MMA runs on the current tile), then
//               layer 1 into the A operand as soon as the MMA has released it.
// Layer 1 is a sparse gather-sum of ~1.6 W1' rows per window (the one-hot input has 64 ones in 448 features
// and ~62 of them are the Fe reference), FP64 on CUDA cores, not a dense GEMM.
#include "akmc_eval.cuh"

namespace akmc {
namespace {
using namespace ptx;

constexpr int kBTile = 128;                                     // rows per tile = TMEM lanes = UMMA M
constexpr int kBEpiWarps = 4;
constexpr int kBLoadWarp = 4, kBMmaWarp = 5;
#ifndef AKMC_BULK_PROD
#define AKMC_BULK_PROD 10       // producer warps (A/B knob): 16 warps in all = 4 per SM sub-partition, 128 registers
#endif
constexpr int kBProdWarp0 = 6, kBProdWarps = AKMC_BULK_PROD;
constexpr int kBThreads = 32 * (kBProdWarp0 + kBProdWarps);    // 512
constexpr int kBStages = 4;
constexpr uint32_t kBSplitA = kBTile * kHid * 2;                // 64 KiB: one fp16 split of the A tile
constexpr uint32_t kBW2Split = kHid * 16 * 2;                   // 8 KiB: one fp16 split of a W2 K-step, N = 256
constexpr uint32_t kBW2Stage = 2 * kBW2Split;                   // hi | lo
constexpr int kBRowsPerProd = (kBTile + kBProdWarps - 1) / kBProdWarps;   // rows pw + P q < 128 of producer pw
static_assert(kBRowsPerProd <= 32, "one lane per row");

struct BulkMeta {                                               // per tile, read by the epilogue
    uint8_t win8[kBTile][8];                                    // first-shell bytes (masks)
    int slot[kBTile];                                           // output index, -1 = padding row
    int vox[kBTile];                                            // voxel (kT_v), -1 = configured T
};

constexpr uint32_t kBOffA = 0;
constexpr uint32_t kBOffRing = kBOffA + 2 * kBSplitA;
constexpr uint32_t kBOffW3 = kBOffRing + kBStages * kBW2Stage;   // double [256][8]
constexpr uint32_t kBOffB1 = kBOffW3 + kHid * 8 * 8;             // float [256]: b1'
constexpr uint32_t kBOffB2 = kBOffB1 + kHid * 4;                 // float [256]
constexpr uint32_t kBOffB3 = kBOffB2 + kHid * 4;                 // double [8]
constexpr uint32_t kBOffWin = kBOffB3 + 8 * 8;                   // uint8 [128][64] (producers)
constexpr uint32_t kBOffL1N = kBOffWin + kBTile * kWin;          // uint8 [128]
constexpr uint32_t kBOffL1L = kBOffL1N + kBTile;                 // uint16 [128][kL1List]
constexpr uint32_t kBOffMeta = (kBOffL1L + kBTile * kL1List * 2 + 15u) & ~15u;   // BulkMeta [2]
constexpr uint32_t kBOffBar = (kBOffMeta + 2 * (uint32_t)sizeof(BulkMeta) + 7u) & ~7u;
// barriers: ring full[4] empty[4], a_full, a_empty, d_full, d_empty, meta_full[2], meta_empty[2]
constexpr int kBNumBars = 2 * kBStages + 8;
constexpr uint32_t kBOffTmem = kBOffBar + kBNumBars * 8;
constexpr uint32_t kBSmemTotal = kBOffTmem + 16 + 128;           // + 128-B alignment slack
static_assert(kBSmemTotal <= 232448, "bulk evaluator shared memory budget");
static_assert(kBOffRing % 128 == 0 && kBOffW3 % 16 == 0 && kBOffMeta % 16 == 0, "alignment");

__global__ void __launch_bounds__(kBThreads, 1) bulk_eval_kernel(const __grid_constant__ BulkParams p)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint8_t* A_hi = sm + kBOffA;
    uint8_t* A_lo = sm + kBOffA + kBSplitA;
    double* w3s = reinterpret_cast<double*>(sm + kBOffW3);
    float* b1s = reinterpret_cast<float*>(sm + kBOffB1);
    float* b2s = reinterpret_cast<float*>(sm + kBOffB2);
    double* b3s = reinterpret_cast<double*>(sm + kBOffB3);
    uint8_t* win = sm + kBOffWin;
    uint8_t* l1n = sm + kBOffL1N;
    uint16_t* l1l = reinterpret_cast<uint16_t*>(sm + kBOffL1L);
    BulkMeta* meta = reinterpret_cast<BulkMeta*>(sm + kBOffMeta);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kBOffBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kBOffTmem);
    const uint32_t bar_full = smem_u32(&bars[0]), bar_empty = smem_u32(&bars[kBStages]);
    const uint32_t bar_afull = smem_u32(&bars[2 * kBStages + 0]), bar_aempty = smem_u32(&bars[2 * kBStages + 1]);
    const uint32_t bar_dfull = smem_u32(&bars[2 * kBStages + 2]), bar_dempty = smem_u32(&bars[2 * kBStages + 3]);
    const uint32_t bar_mfull = smem_u32(&bars[2 * kBStages + 4]), bar_mempty = smem_u32(&bars[2 * kBStages + 6]);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool fast = p.fast != 0;

    const int nrows = p.nrows_dev ? *p.nrows_dev : p.nrows_host;
    const int ntiles = (nrows + kBTile - 1) / kBTile;

    if (tid == 0) {
        for (int s = 0; s < kBStages; ++s) { mbar_init(bar_full + 8 * s, 1); mbar_init(bar_empty + 8 * s, 1); }
        mbar_init(bar_afull, kBProdWarps);
        mbar_init(bar_aempty, 1);
        mbar_init(bar_dfull, 1);
        mbar_init(bar_dempty, kBEpiWarps);
        for (int b = 0; b < 2; ++b) { mbar_init(bar_mfull + 8 * b, kBProdWarps); mbar_init(bar_mempty + 8 * b, kBEpiWarps); }
        mbar_fence_init();
    }
    for (int i = tid; i < kHid * 8; i += kBThreads) w3s[i] = p.W.W3d[i];
    for (int i = tid; i < kHid; i += kBThreads) { b1s[i] = p.W.W1f[i]; b2s[i] = p.W.b2[i]; }
    if (tid < 8) b3s[tid] = p.W.b3[tid];
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    unsigned long long ovf = 0;

    if (warp == kBLoadWarp) {
        // ---------------- W2 loader: the K-steps of every tile through the ring
        if (lane == 0) {
            uint32_t st = 0, ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
                for (int ks = 0; ks < kHid / 16; ++ks) {
                    mbar_wait(bar_empty + 8 * st, ph ^ 1u);
                    mbar_expect_tx(bar_full + 8 * st, kBW2Stage);
                    bulk_g2s(smem_u32(sm + kBOffRing + st * kBW2Stage), p.W2full + (size_t)ks * kBW2Stage, kBW2Stage,
                             bar_full + 8 * st);
                    if (++st == kBStages) { st = 0; ph ^= 1u; }
                }
        }
    } else if (warp == kBMmaWarp) {
        // ---------------- MMA issuer
        if (lane == 0) {
            uint32_t st = 0, ph = 0;
            const uint32_t idesc = idesc_f16(kBTile, kHid);
            const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo);
            int i = 0;
            long long ta = 0, td = 0, tk = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                long long t0 = clock64();
                mbar_wait(bar_afull, (uint32_t)i & 1u);
                long long t1 = clock64(); ta += t1 - t0; t0 = t1;
                if (i > 0) mbar_wait(bar_dempty, (uint32_t)(i - 1) & 1u);
                t1 = clock64(); td += t1 - t0; t0 = t1;
                tc_fence_after();
                for (int ks = 0; ks < kHid / 16; ++ks) {
                    mbar_wait(bar_full + 8 * st, ph);
                    tc_fence_after();
                    const uint32_t wb = smem_u32(sm + kBOffRing + st * kBW2Stage);
                    const uint64_t dah = umma_desc(ah + (uint32_t)ks * 256u, 128, kRowGroupA);
                    const uint64_t dal = umma_desc(al + (uint32_t)ks * 256u, 128, kRowGroupA);
                    const uint64_t dbh = umma_desc(wb, (kHid / 8) * 128, 128);
                    const uint64_t dbl = umma_desc(wb + kBW2Split, (kHid / 8) * 128, 128);
                    umma_f16(tmem + 0, dah, dbh, idesc, ks > 0 ? 1u : 0u);
                    if (!fast) {
                        umma_f16(tmem + kHid, dah, dbl, idesc, ks > 0 ? 1u : 0u);
                        umma_f16(tmem + kHid, dal, dbh, idesc, 1u);
                    }
                    umma_commit(bar_empty + 8 * st);          // the stage is free once these MMAs completed
                    if (++st == kBStages) { st = 0; ph ^= 1u; }
                }
                umma_commit(bar_aempty);                      // A may be overwritten
                umma_commit(bar_dfull);                       // accumulators complete
                tk += clock64() - t0;
            }
            if (p.diag) {
                atomicAdd(p.diag + 5, (unsigned long long)ta); atomicAdd(p.diag + 6, (unsigned long long)td);
                atomicAdd(p.diag + 7, (unsigned long long)tk); atomicAdd(p.diag + 8, (unsigned long long)i);
            }
        }
    } else if (warp >= kBProdWarp0) {
        // ---------------- producers: gather (overlaps the previous tile's MMA), then layer 1 into A
        const int pw = warp - kBProdWarp0;
        const uint32_t off_lo = pack_off(p.G.off[lane]), off_hi = pack_off(p.G.off[lane + 32]);
        long long tg = 0, tw = 0, tl = 0, tm = 0;          // diag: gather, wait A, layer 1, wait meta
        int i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int b = i & 1;
            long long t0 = clock64();
            if (i >= 2) mbar_wait(bar_mempty + 8 * b, (uint32_t)((i >> 1) - 1) & 1u);
            long long t1 = clock64(); tm += t1 - t0; t0 = t1;
            BulkMeta& M = meta[b];
            // rows pw + 8 q (q = 0..15): lane q < 16 resolves row q's source (slot, position), then all 32 window
            // bytes of the lane's two slots for the 16 rows are in flight at once
            int my_slot = -1, my_vox = -1;
            int4 my_v = make_int4(-1, 0, 0, 0);
            const bool row_ok = lane < kBRowsPerProd && pw + kBProdWarps * lane < kBTile;
            if (row_ok) {
                const int g = t * kBTile + pw + kBProdWarps * lane;
                if (g < nrows) {
                    if (p.windows) {
                        my_slot = g;
                    } else {
                        my_slot = p.rows ? p.rows[g] : g;
                        my_v = p.vac[my_slot];
                        my_vox = max(my_v.x, 0);
                    }
                }
            }
            uint8_t b0[kBRowsPerProd], b1[kBRowsPerProd];
#pragma unroll
            for (int q = 0; q < kBRowsPerProd; ++q) {
                const int sl = __shfl_sync(0xffffffffu, my_slot, q);
                int4 v;
                v.x = __shfl_sync(0xffffffffu, my_v.x, q); v.y = __shfl_sync(0xffffffffu, my_v.y, q);
                v.z = __shfl_sync(0xffffffffu, my_v.z, q); v.w = __shfl_sync(0xffffffffu, my_v.w, q);
                b0[q] = (uint8_t)kFe; b1[q] = (uint8_t)kFe;
                if (sl >= 0) {
                    if (p.windows) {
                        b0[q] = p.windows[(size_t)sl * kWin + lane];
                        b1[q] = p.windows[(size_t)sl * kWin + lane + 32];
                    } else if (v.x >= 0) {                       // departed slot (multi-rank): any window
                        b0[q] = site_byte_pk(p.species, p.F, v, off_lo);
                        b1[q] = site_byte_pk(p.species, p.F, v, off_hi);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kBRowsPerProd; ++q) {
                const int r = pw + kBProdWarps * q;
                if (kBTile % kBProdWarps != 0 && r >= kBTile) break;   // warp-uniform
                win[r * kWin + lane] = b0[q];
                win[r * kWin + lane + 32] = b1[q];
                if (lane < 8) M.win8[r][lane] = b0[q];
                l1_list_store(r, b0[q], b1[q], l1n, l1l);
            }
            if (row_ok) {
                const int r = pw + kBProdWarps * lane;
                M.slot[r] = my_slot;
                M.vox[r] = my_vox;
            }
            __syncwarp();
            t1 = clock64(); tg += t1 - t0; t0 = t1;
            // layer 1 needs the A operand released by the previous tile's MMAs
            if (i > 0) mbar_wait(bar_aempty, (uint32_t)(i - 1) & 1u);
            t1 = clock64(); tw += t1 - t0; t0 = t1;
#pragma unroll 1
            for (int q0 = 0; q0 < kBRowsPerProd; q0 += kL1Rows) {
                int rr[kL1Rows], mr[kL1Rows], nv = 0;
#pragma unroll
                for (int q = 0; q < kL1Rows; ++q) {
                    rr[q] = pw + kBProdWarps * (q0 + q);
                    if (q0 + q < kBRowsPerProd && rr[q] < kBTile) ++nv; else rr[q] = 0;   // (valid rows first)
                    mr[q] = rr[q];
                }
                layer1_rows(rr, nv, win, l1n, l1l, p.W.W1f, mr, A_hi, A_lo, nullptr, nullptr, ovf, fast, p.W.h1s,
                            nullptr, b1s);
            }
            fence_async_smem();                                 // generic-proxy A writes -> the MMA's async proxy
            __syncwarp();
            if (lane == 0) { mbar_arrive(bar_afull); mbar_arrive(bar_mfull + 8 * b); }
            tl += clock64() - t0;
        }
        if (p.diag && lane == 0) {
            atomicAdd(p.diag + 0, (unsigned long long)tg); atomicAdd(p.diag + 1, (unsigned long long)tw);
            atomicAdd(p.diag + 2, (unsigned long long)tl); atomicAdd(p.diag + 3, (unsigned long long)tm);
            atomicAdd(p.diag + 4, 1ull);
        }
    } else {
        // ---------------- epilogue warps 0-3: row m = TMEM lane 32 w + lane
        const int m = 32 * warp + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);
        long long tw = 0, tc = 0, te = 0;
        int i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int b = i & 1;
            long long t0 = clock64();
            mbar_wait(bar_dfull, (uint32_t)i & 1u);
            mbar_wait(bar_mfull + 8 * b, (uint32_t)(i >> 1) & 1u);
            long long t1 = clock64(); tw += t1 - t0; t0 = t1;
            tc_fence_after();
            double acc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = 0.0;
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
                double pa[8], Sr[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int q = 4 * r + j;
                    uint32_t d1[16], d2[16];
                    tmem_ld16(tl + (uint32_t)(16 * q), d1);
                    if (!fast) tmem_ld16(tl + (uint32_t)(kHid + 16 * q), d2);
                    else
#pragma unroll
                        for (int u = 0; u < 16; ++u) d2[u] = 0u;
                    tmem_wait_ld();
                    float z[16];
                    e2_chunk(d1, d2, b2s + 16 * q, p.W.s2u, z);
                    double P[8];
                    l3_chunk(z, w3s + 16 * q * 8, P);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (j == 0 || j == 2) pa[k] = P[k];
                        else if (j == 1) Sr[k] = __dadd_rn(pa[k], P[k]);
                        else Sr[k] = __dadd_rn(Sr[k], __dadd_rn(pa[k], P[k]));
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = __dadd_rn(acc[k], Sr[k]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_dempty);            // TMEM may be overwritten by the next tile
            t1 = clock64(); tc += t1 - t0; t0 = t1;
            const int slot = meta[b].slot[m];
            if (slot >= 0) {
                const int vox = meta[b].vox[m];
                double R = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double out = __dadd_rn(b3s[k], acc[k]);
                    const double Ek = out > 0.0 ? out : 0.0;
                    const double g = arrhenius_tc(Ek, p.P, vox);   // unconditional: the 8 exps run interleaved
                    const double Gk = (meta[b].win8[m][k] != (uint8_t)kVac) ? g : 0.0;
                    R = __dadd_rn(R, Gk);
                    if (p.rates) p.rates[(size_t)slot * 8 + k] = Gk;
                    if (p.E) p.E[(size_t)slot * 8 + k] = Ek;
                }
                if (p.Rsum) p.Rsum[slot] = R;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_mempty + 8 * b);
            te += clock64() - t0;
        }
        if (p.diag && lane == 0) {
            atomicAdd(p.diag + 9, (unsigned long long)tw); atomicAdd(p.diag + 10, (unsigned long long)tc);
            atomicAdd(p.diag + 11, (unsigned long long)te); atomicAdd(p.diag + 12, 1ull);
        }
    }
    if (ovf && p.overflow) atomicAdd(p.overflow, ovf);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

} // namespace

cudaError_t bulk_setup()
{
    return cudaFuncSetAttribute(bulk_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmemTotal);
}

cudaError_t launch_bulk(const BulkParams& p, int max_rows, int num_sms, cudaStream_t s)
{
    const int tiles = (max_rows + kBTile - 1) / kBTile;
    const int grid = std::max(1, std::min(num_sms, tiles));
    bulk_eval_kernel<<<grid, kBThreads, kBSmemTotal, s>>>(p);
    return cudaGetLastError();
}

} // namespace akmc
