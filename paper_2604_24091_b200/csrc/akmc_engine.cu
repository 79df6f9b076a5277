// akmc_engine.cu -- sublattice phase engine (see akmc_engine.cuh) and its barrier-network evaluator.
//
// Control (every CTA, independently): hold up to 16 domains (segments) of the current phase; per
// iteration gather the 64-site window of every active vacancy, look the window up in the
// per-vacancy memo, evaluate the misses, then run one BKL step per running domain (tree over the
// domain's rates, Philox draw, window test, hop) exactly as the oracle's run_sublattice does; refill
// from the phase's segment list when all held domains have stopped.
//
// Evaluator, FP32-equivalent mode (cluster of 8 CTAs, rounds in lockstep): each CTA contributes up to
// 16 miss rows per round (tile M = 128 rows = 8 x 16) and broadcasts their windows to the cluster;
//   L1 (CUDA cores): CTA r computes h1[:, 32r:32r+32] = ReLU(b1' + sum over the row's non-Fe slots of
//      W1'(s, slot)) -- the one-hot layer is a sparse gather-sum (~6 terms), not a dense contraction --
//      in FP64, rounded once to FP32 and split into fp16 hi + lo*2^-11; the slice is bulk-copied into
//      the A operand of the other 7 CTAs (DSMEM);
//   L2 (tcgen05, M=128 N=32 K=256): D1 = Ahi*W2hi, D2 = Ahi*W2lo + Alo*W2hi with CTA r's resident
//      W2 slice; h2 = ReLU(2^-s2 (D1 + 2^-11 D2) + b2) -> fp16 split (local);
//   L3 (tcgen05, M=128 N=16 K=32): CTA r's partial of the 8 outputs over its 32 h2 columns; the
//      partials of row block [16s, 16s+16) are bulk-copied to CTA s, which sums them in fixed order
//      (FP64), adds b3, clamps at 0 and forms Gamma = nu0 det_exp(-E/kT).
// The result of a row depends only on its window (rows of a tile do not interact, the order of every
// sum is fixed), so memoisation and any tiling or decomposition give bit-identical trajectories.
// FP64 verify mode: each CTA evaluates its own misses (pair KRA or FP64 MLP, same code as the FP64
// kernels), no cluster.
#include "akmc_engine.cuh"
#include "akmc_ptx.cuh"

namespace akmc {

namespace {
using namespace ptx;

constexpr int kThreads = 256;
constexpr int kTileRows = kRoundRows * kClusterN;              // 128
constexpr uint32_t kCoreCol = (kTileRows / 8) * 128;           // 2048 B between K-adjacent core matrices
constexpr uint32_t kSplitA = kTileRows * kHid * 2;             // 64 KiB: one fp16 split of h1
constexpr uint32_t kSplitH2 = kTileRows * kSliceN * 2;         // 8 KiB: one fp16 split of the h2 slice
constexpr uint32_t kW2Split = kSliceN * 16 * 2;                // 1 KiB: one split of a W2-slice K-step
constexpr uint32_t kW2Bytes = (kHid / 16) * 2 * kW2Split;      // 32 KiB
constexpr uint32_t kW3Split = 16 * 16 * 2;                     // 512 B
constexpr uint32_t kW3Bytes = (kSliceN / 16) * 2 * kW3Split;   // 2 KiB
constexpr uint32_t kReqBytes = 16 + kRoundRows * kWin;         // header + 16 windows
constexpr float kLo = 2048.0f;

struct ReqHdr { int n, more, alive, pad; };

struct Ctl {
    long long seg_dom[kSegsPerCta];
    double seg_t[kSegsPerCta];
    int seg_goff[kSegsPerCta];      // global member offset (scratch of big trees)
    int seg_moff[kSegsPerCta];      // offset into the CTA's member arrays
    int seg_cnt[kSegsPerCta];
    unsigned seg_it[kSegsPerCta];
    int seg_run[kSegsPerCta];
    long long cand_dom[2 * kSegsPerCta];   // domains waiting to be loaded: [0, npend) carried over, then new
    int cand_off[2 * kSegsPerCta];
    int cand_cnt[2 * kSegsPerCta];
    int npend, ncand, refill, drained, ntot, s0;
    int nseg, nmem, nrows, nmiss, nrun, ebase;
    int wsum[8];
    int4 mem_vac[kRowCap];          // positions of the held vacancies (this CTA is their only writer)
    int mem_slot[kRowCap];
    short mem_row[kRowCap];
    short row_mem[kRowCap];
    short miss[kRowCap];
    uint8_t mem_act[kRowCap];
    uint8_t mem_seg[kRowCap];
    uint8_t row_hit[kRowCap];
    unsigned long long events, evals, mrows, clamps;
};

// shared-memory carve-up (offsets from a 1024-aligned base)
constexpr uint32_t kOffA = 0;                                        // h1 hi [0,64K) lo [64K,128K); FP64 scratch
constexpr uint32_t kOffH2 = kOffA + 2 * kSplitA;                     // h2 hi/lo | layer-1 lists | partials out
constexpr uint32_t kOffW2 = kOffH2 + 2 * kSplitH2;
constexpr uint32_t kOffW3 = kOffW2 + kW2Bytes;
constexpr uint32_t kOffReq = kOffW3 + kW3Bytes;                      // [8 sources][kReqBytes]
constexpr uint32_t kOffPart = kOffReq + kClusterN * kReqBytes;       // [8 sources][16 rows][8] double
constexpr uint32_t kOffWin = kOffPart + kClusterN * kRoundRows * 8 * 8;   // own rows' windows [128][64]
constexpr uint32_t kOffRowG = kOffWin + kRowCap * kWin;              // [128][8] double
constexpr uint32_t kOffRowR = kOffRowG + kRowCap * 8 * 8;            // [128] double
constexpr uint32_t kOffRowC = kOffRowR + kRowCap * 8;                // [128] int
constexpr uint32_t kOffB2 = kOffRowC + kRowCap * 4;                  // float [32]
constexpr uint32_t kOffB3 = kOffB2 + kSliceN * 4;                    // double [8]
constexpr uint32_t kOffNl = kOffB3 + 8 * 8;                          // uint8 [128] layer-1 list lengths
constexpr uint32_t kOffCtl = kOffNl + kTileRows;
constexpr uint32_t kOffBar = (kOffCtl + (uint32_t)sizeof(Ctl) + 7u) & ~7u;
constexpr int kNumBars = 5;                                          // req, h1, part, mma, weights
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemUsed = kOffTmem + 16;
constexpr uint32_t kSmemTotal = kSmemUsed + 1024;
static_assert(kSmemTotal <= 232448, "shared memory budget");
static_assert(kOffReq % 16 == 0 && kOffPart % 16 == 0 && kOffW2 % 16 == 0 && kOffW3 % 16 == 0, "bulk alignment");
static_assert(kReqBytes % 16 == 0, "bulk size");
static_assert(kRoundRows * kWin * 2 * 8 <= 2 * kSplitH2, "layer-1 lists fit the h2 region");

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive block prefix of v over threads [0, 256); returns prefix, *total gets the sum (all threads)
__device__ __forceinline__ int block_excl(int v, int* wsum, int& total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int base = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const int t = wsum[w];
        if (w < wid) base += t;
        total += t;
    }
    return base + incl - v;
}

// fp16 hi/lo split of an FP32 value (lo carries the remainder * 2^11)
__device__ __forceinline__ void split_h(float v, __half& hi, __half& lo, unsigned long long& ovf)
{
    if (v > 60000.0f) { v = 60000.0f; ++ovf; }
    hi = __float2half_rn(v);
    lo = __float2half_rn((v - __half2float(hi)) * kLo);
}

// no-swizzle K-major operand offset of element (m, k) in a 128-row tile
__device__ __forceinline__ uint32_t kmaj_off(int m, int k)
{
    return (uint32_t)(k >> 3) * kCoreCol + (uint32_t)(m >> 3) * 128u + (uint32_t)(m & 7) * 16u + (uint32_t)(k & 7) * 2u;
}

// window byte loads of an owned vacancy: plain (coherent) loads -- the lattice is written by this kernel
__device__ __forceinline__ uint8_t site_byte(const uint8_t* species, const Frame& F, const int4& v, const int8_t* o)
{
    return species[neighbour_site(F, v, o[0], o[1], o[2])];
}

template <bool kTC>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ EngineParams p)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    Ctl& c = *reinterpret_cast<Ctl*>(sm + kOffCtl);
    uint8_t* win = sm + kOffWin;
    double* rowG = reinterpret_cast<double*>(sm + kOffRowG);
    double* rowR = reinterpret_cast<double*>(sm + kOffRowR);
    int* rowC = reinterpret_cast<int*>(sm + kOffRowC);
    uint8_t* A_hi = sm + kOffA;
    uint8_t* A_lo = sm + kOffA + kSplitA;
    uint8_t* H2_hi = sm + kOffH2;
    uint8_t* H2_lo = sm + kOffH2 + kSplitH2;
    uint16_t* lists = reinterpret_cast<uint16_t*>(sm + kOffH2);     // [128][64] (layer 1 only)
    double* part_out = reinterpret_cast<double*>(sm + kOffH2);      // [128][8]  (after layer 3)
    double* part_in = reinterpret_cast<double*>(sm + kOffPart);     // [8][16][8]
    uint8_t* nl = sm + kOffNl;
    float* b2s = reinterpret_cast<float*>(sm + kOffB2);
    double* b3s = reinterpret_cast<double*>(sm + kOffB3);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kOffTmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = kTC ? cluster_rank() : 0u;
    const uint32_t bar_req = smem_u32(&bars[0]), bar_h1 = smem_u32(&bars[1]), bar_part = smem_u32(&bars[2]);
    const uint32_t bar_mma = smem_u32(&bars[3]), bar_w = smem_u32(&bars[4]);
    const bool phase_mode = (p.mode == kEnginePhase);
    const bool mlp = (p.model == 1);
    unsigned long long ovf = 0;

    if (tid == 0) {
        c.nseg = 0; c.npend = 0; c.drained = 0; c.nmem = 0; c.nrun = 0;
        c.ntot = phase_mode ? (int)p.ctr->nseg : 0;
        c.events = 0; c.evals = 0; c.mrows = 0; c.clamps = 0;
        if (kTC) {
            mbar_init(bar_req, kClusterN);
            mbar_init(bar_h1, kClusterN - 1);
            mbar_init(bar_part, kClusterN);
            mbar_init(bar_mma, 1);
            mbar_init(bar_w, 1);
            mbar_fence_init();
        }
    }
    uint32_t tmem = 0;
    uint32_t ph_req = 0, ph_h1 = 0, ph_part = 0, ph_mma = 0;
    if (kTC) {
        if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 128);
        if (tid < kSliceN) b2s[tid] = p.W.b2[rank * kSliceN + tid];
        if (tid < 8) b3s[tid] = p.W.b3[tid];
        tc_fence_before();
        cluster_sync();                            // every barrier of the cluster initialised
        tc_fence_after();
        tmem = *tmem_slot;
        if (tid == 0) {
            mbar_expect_tx(bar_w, kW2Bytes + kW3Bytes);
            bulk_g2s(smem_u32(sm + kOffW2), p.W.W2img + (size_t)rank * kW2Bytes, kW2Bytes, bar_w);
            bulk_g2s(smem_u32(sm + kOffW3), p.W.W3img + (size_t)rank * kW3Bytes, kW3Bytes, bar_w);
        }
        mbar_wait(bar_w, 0);
    } else {
        __syncthreads();
    }
    const int nrows_eval = (!phase_mode) ? (p.nrows_dev ? *p.nrows_dev : p.nrows_host) : 0;

    for (;;) {
        // ================= control: refill, rows, gather + memo lookup =================
        int own_alive = 0;
        if (phase_mode) {
            // ---- refill when every held domain has stopped: carried-over domains first, then the next
            //      kSegsPerCta entries of the phase's segment list (domains are independent: any order)
            __syncthreads();
            if (tid == 0) {
                c.refill = (c.nrun == 0) ? 1 : 0;
                c.ncand = c.npend;
                if (c.refill && c.npend == 0 && !c.drained) {
                    const int s0 = (int)atomicAdd(&p.ctr->chunk, (unsigned long long)kSegsPerCta);
                    if (s0 >= c.ntot) c.drained = 1;
                    else { c.s0 = s0; c.ncand = min(kSegsPerCta, c.ntot - s0); }
                }
            }
            __syncthreads();
            if (c.refill && c.npend == 0 && tid < c.ncand) {
                const Segment sg = p.segs[c.s0 + tid];
                c.cand_dom[tid] = sg.dom; c.cand_off[tid] = sg.off; c.cand_cnt[tid] = sg.cnt;
            }
            __syncthreads();
            if (tid == 0 && c.refill) {
                int nseg = 0, nmem = 0, np = 0;
                for (int q = 0; q < c.ncand; ++q) {
                    const int cnt = c.cand_cnt[q];
                    if (cnt > kRowCap) { atomicAdd(p.overflow, 1ull); continue; }   // can never be held
                    if (nseg < kSegsPerCta && nmem + cnt <= kRowCap) {
                        c.seg_dom[nseg] = c.cand_dom[q]; c.seg_goff[nseg] = c.cand_off[q]; c.seg_cnt[nseg] = cnt;
                        c.seg_moff[nseg] = nmem; c.seg_t[nseg] = 0.0; c.seg_it[nseg] = 0u; c.seg_run[nseg] = 1;
                        nmem += cnt;
                        ++nseg;
                    } else {                                   // carried over (np <= q: in-place is safe)
                        c.cand_dom[np] = c.cand_dom[q]; c.cand_off[np] = c.cand_off[q]; c.cand_cnt[np] = cnt;
                        ++np;
                    }
                }
                c.npend = np; c.nseg = nseg; c.nmem = nmem; c.nrun = nseg;
            }
            __syncthreads();
            if (c.refill) {
                for (int i = warp; i < c.nseg; i += kThreads / 32) {
                    const int cnt = c.seg_cnt[i], moff = c.seg_moff[i], goff = c.seg_goff[i];
                    for (int a = lane; a < cnt; a += 32) {
                        const int slot = p.members[goff + a];
                        c.mem_slot[moff + a] = slot;
                        c.mem_vac[moff + a] = p.vac[slot];
                        c.mem_act[moff + a] = 1;
                        c.mem_seg[moff + a] = (uint8_t)i;
                    }
                }
            }
            __syncthreads();
            own_alive = c.nrun > 0 ? 1 : 0;
            // rows = active members of running domains, in member order
            int total = 0;
            {
                const int pidx = tid;
                const bool act = pidx < c.nmem && c.mem_act[pidx] && c.seg_run[c.mem_seg[pidx]];
                const int r = block_excl(act ? 1 : 0, c.wsum, total);
                if (pidx < kRowCap) c.mem_row[pidx] = act ? (short)r : (short)-1;
                if (act) c.row_mem[r] = (short)pidx;
            }
            if (tid == 0) c.nrows = total;
            __syncthreads();
            // gather + memo: warp per row, lane = window slots j and j+32
            const int nrows = c.nrows;
            for (int r = warp; r < nrows; r += kThreads / 32) {
                const int slot = c.mem_slot[c.row_mem[r]];
                const int4 v = c.mem_vac[c.row_mem[r]];
                const MemoEntry* me = p.memo + 2 * (size_t)slot;
                const uint32_t kw = reinterpret_cast<const uint32_t*>(me[lane >> 4].key)[lane & 15];
                double gv = 0.0;
                int cv = 0;
                {
                    const int k = lane & 15;
                    const MemoEntry& e = me[lane >> 4];
                    if (k < 8) gv = e.G[k];
                    else if (k == 8) gv = e.R;
                    else if (k == 9) cv = e.clamps;
                }
                const uint8_t b0 = site_byte(p.species, p.F, v, p.G.off[lane]);
                const uint8_t b1 = site_byte(p.species, p.F, v, p.G.off[lane + 32]);
                win[r * kWin + lane] = b0;
                win[r * kWin + lane + 32] = b1;
                __syncwarp();
                const uint32_t ww = reinterpret_cast<const uint32_t*>(win + r * kWin)[lane & 15];
                const unsigned eq = __ballot_sync(0xffffffffu, ww == kw);
                const int hit = (eq & 0xFFFFu) == 0xFFFFu ? 0 : ((eq >> 16) == 0xFFFFu ? 1 : -1);
                if (hit >= 0 && (lane >> 4) == hit) {
                    const int k = lane & 15;
                    if (k < 8) rowG[r * 8 + k] = gv;
                    else if (k == 8) rowR[r] = gv;
                    else if (k == 9) rowC[r] = cv;
                }
                if (lane == 0) c.row_hit[r] = hit >= 0 ? 1 : 0;
            }
            __syncthreads();
            {
                const bool ms = tid < nrows && !c.row_hit[tid];
                const int q = block_excl(ms ? 1 : 0, c.wsum, total);
                if (ms) c.miss[q] = (short)tid;
            }
            if (tid == 0) { c.nmiss = total; c.mrows += (unsigned long long)total; }
            __syncthreads();
        }

        // ================= evaluation of the misses =================
        bool all_dead = false;
        if (!kTC) {
            if (!own_alive) break;
            const int nmiss = c.nmiss;
            if (!mlp) {
                for (int q = tid; q < nmiss; q += kThreads) {
                    const int r = c.miss[q];
                    const uint8_t* w = win + r * kWin;
                    double R = 0.0;
                    int cl = 0;
                    for (int k = 0; k < kHops; ++k) {
                        double E = 0.0, Gk = 0.0;
                        if (w[k] != kVac) {
                            cl += pair_barrier(w, k, p.G, p.P, E);
                            Gk = arrhenius(E, p.P);
                        }
                        R = __dadd_rn(R, Gk);
                        rowG[r * 8 + k] = Gk;
                    }
                    rowR[r] = R;
                    rowC[r] = cl;
                }
            } else {
                double* h1 = reinterpret_cast<double*>(sm + kOffA);
                double* h2 = h1 + kHid;
                double* Ek = h2 + kHid;
                const double* W1 = p.W.mlp64;
                const double* b1 = W1 + 448 * kHid;
                const double* W2 = b1 + kHid;
                const double* b2 = W2 + kHid * kHid;
                const double* W3 = b2 + kHid;
                const double* b3 = W3 + kHid * 8;
                const int j = tid;
                for (int q = 0; q < nmiss; ++q) {
                    const int r = c.miss[q];
                    const uint8_t* w = win + r * kWin;
                    double acc = b1[j];
                    for (int s = 0; s < kWin; ++s) acc = __dadd_rn(acc, W1[(size_t)(kSpecies * s + w[s]) * kHid + j]);
                    h1[j] = acc > 0.0 ? acc : 0.0;
                    __syncthreads();
                    acc = b2[j];
                    for (int i = 0; i < kHid; ++i) acc = __fma_rn(h1[i], W2[(size_t)i * kHid + j], acc);
                    h2[j] = acc > 0.0 ? acc : 0.0;
                    __syncthreads();
                    if (j < 8) {
                        acc = b3[j];
                        for (int i = 0; i < kHid; ++i) acc = __fma_rn(h2[i], W3[i * 8 + j], acc);
                        Ek[j] = acc > 0.0 ? acc : 0.0;
                    }
                    __syncthreads();
                    if (j == 0) {
                        double R = 0.0;
                        for (int k = 0; k < kHops; ++k) {
                            const double Gk = (w[k] != kVac) ? arrhenius(Ek[k], p.P) : 0.0;
                            R = __dadd_rn(R, Gk);
                            rowG[r * 8 + k] = Gk;
                        }
                        rowR[r] = R;
                        rowC[r] = 0;
                    }
                    __syncthreads();
                }
            }
            __syncthreads();
            // memo insert: way 1 <- way 0, way 0 <- (window, rates)
            for (int q = warp; q < nmiss; q += kThreads / 32) {
                const int r = c.miss[q];
                MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                uint4* d1 = reinterpret_cast<uint4*>(&me[1]);
                const uint4* s0 = reinterpret_cast<const uint4*>(&me[0]);
                uint4 t = make_uint4(0, 0, 0, 0);
                if (lane < 9) t = s0[lane];
                __syncwarp();
                if (lane < 9) d1[lane] = t;
                __syncwarp();
                if (lane < 16) reinterpret_cast<uint32_t*>(me[0].key)[lane] = reinterpret_cast<const uint32_t*>(win + r * kWin)[lane];
                else if (lane < 24) me[0].G[lane - 16] = rowG[r * 8 + lane - 16];
                else if (lane == 24) me[0].R = rowR[r];
                else if (lane == 25) me[0].clamps = rowC[r];
            }
        } else {
            // ---- FP32-equivalent evaluator: rounds in lockstep over the cluster
            int k_round = 0;
            for (;;) {
                uint8_t* req_own = sm + kOffReq + rank * kReqBytes;
                ReqHdr* hdr_own = reinterpret_cast<ReqHdr*>(req_own);
                uint8_t* wreq = req_own + 16;
                int own_n = 0;
                if (phase_mode) {
                    const int nmiss = c.nmiss;
                    own_n = min(kRoundRows, max(0, nmiss - kRoundRows * k_round));
                    // own request: windows of misses [16k, 16k+16); memo way 1 <- way 0, way 0 key <- window
                    {
                        const int i = tid >> 4, wd = tid & 15;
                        if (i < own_n) {
                            const int r = c.miss[kRoundRows * k_round + i];
                            reinterpret_cast<uint32_t*>(wreq + i * kWin)[wd] = reinterpret_cast<const uint32_t*>(win + r * kWin)[wd];
                        }
                    }
                    for (int i = warp; i < own_n; i += kThreads / 32) {
                        const int r = c.miss[kRoundRows * k_round + i];
                        MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                        uint4 t = make_uint4(0, 0, 0, 0);
                        if (lane < 9) t = reinterpret_cast<const uint4*>(&me[0])[lane];
                        __syncwarp();
                        if (lane < 9) reinterpret_cast<uint4*>(&me[1])[lane] = t;
                        __syncwarp();
                        if (lane < 16) reinterpret_cast<uint32_t*>(me[0].key)[lane] = reinterpret_cast<const uint32_t*>(win + r * kWin)[lane];
                    }
                    if (tid == 0) {
                        hdr_own->n = own_n;
                        hdr_own->more = (c.nmiss > kRoundRows * (k_round + 1)) ? 1 : 0;
                        hdr_own->alive = own_alive;
                    }
                } else {
                    // eval mode: the next 16 rows from the cursor
                    __syncthreads();
                    if (tid == 0) c.ebase = (int)atomicAdd(p.cursor, (unsigned)kRoundRows);
                    __syncthreads();
                    const int base = c.ebase;
                    own_n = min(kRoundRows, max(0, nrows_eval - base));
                    for (int i = warp; i < own_n; i += kThreads / 32) {
                        const int g = base + i;
                        if (p.windows) {
                            wreq[i * kWin + lane] = p.windows[(size_t)g * kWin + lane];
                            wreq[i * kWin + lane + 32] = p.windows[(size_t)g * kWin + lane + 32];
                        } else {
                            const int slot = p.rows ? p.rows[g] : g;
                            const int4 v = p.vac[slot];
                            wreq[i * kWin + lane] = site_byte(p.species, p.F, v, p.G.off[lane]);
                            wreq[i * kWin + lane + 32] = site_byte(p.species, p.F, v, p.G.off[lane + 32]);
                        }
                    }
                    if (tid == 0) { hdr_own->n = own_n; hdr_own->more = 0; hdr_own->alive = own_n > 0 ? 1 : 0; }
                }
                // ---- exchange requests (every CTA sends exactly one per round)
                fence_async_smem();
                __syncthreads();
                if (tid == 0) {
                    for (uint32_t d = 0; d < (uint32_t)kClusterN; ++d) {
                        if (d == rank) continue;
                        const uint32_t cb = map_to(bar_req, d);
                        mbar_remote_expect_tx(cb, kReqBytes);
                        bulk_s2peer(map_to(smem_u32(req_own), d), smem_u32(req_own), kReqBytes, cb);
                    }
                    mbar_arrive(bar_req);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                mbar_wait_cluster(bar_req, ph_req);
                ph_req ^= 1u;
                int n_s[kClusterN];
                int any_more = 0, any_alive = 0, maxrow = 0, total = 0;
#pragma unroll
                for (int s = 0; s < kClusterN; ++s) {
                    const ReqHdr* hs = reinterpret_cast<const ReqHdr*>(sm + kOffReq + s * kReqBytes);
                    n_s[s] = hs->n;
                    any_more |= hs->more;
                    any_alive |= hs->alive;
                    total += hs->n;
                    if (hs->n > 0) maxrow = kRoundRows * s + hs->n;
                }
                if (k_round == 0 && !any_alive) { all_dead = true; }
                if (total > 0) {
                    // ---- L1: layer-1 lists (non-Fe slots in slot order) of all tile rows, warp per row
                    for (int m = warp; m < kTileRows; m += kThreads / 32) {
                        const int s = m >> 4, i = m & 15;
                        if (i >= n_s[s]) continue;
                        const uint8_t* w = sm + kOffReq + s * kReqBytes + 16 + i * kWin;
                        const uint32_t b0 = w[lane], b1 = w[lane + 32];
                        const unsigned m0 = __ballot_sync(0xffffffffu, b0 != (uint32_t)kFe);
                        const unsigned m1 = __ballot_sync(0xffffffffu, b1 != (uint32_t)kFe);
                        const uint32_t lt = lanemask_lt();
                        if (b0 != (uint32_t)kFe) lists[m * kWin + __popc(m0 & lt)] = (uint16_t)(1 + (b0 - 1) * kWin + lane);
                        if (b1 != (uint32_t)kFe) lists[m * kWin + __popc(m0) + __popc(m1 & lt)] = (uint16_t)(1 + (b1 - 1) * kWin + lane + 32);
                        if (lane == 0) nl[m] = (uint8_t)(__popc(m0) + __popc(m1));
                    }
                    __syncthreads();
                    // ---- L1: h1[:, 32r + lane] for the valid rows; FP64 sum in slot order, one FP32 rounding
                    {
                        const int col = (int)rank * kSliceN + lane;
                        const float bias = p.W.W1f[col];
                        for (int m = warp; m < kTileRows; m += kThreads / 32) {
                            const int s = m >> 4, i = m & 15;
                            if (i >= n_s[s]) continue;
                            const int n = nl[m];
                            const uint16_t* L = lists + m * kWin;
                            double acc = (double)bias;
                            int e = 0;
                            for (; e + 4 <= n; e += 4) {
                                const float x0 = p.W.W1f[(size_t)L[e] * kHid + col];
                                const float x1 = p.W.W1f[(size_t)L[e + 1] * kHid + col];
                                const float x2 = p.W.W1f[(size_t)L[e + 2] * kHid + col];
                                const float x3 = p.W.W1f[(size_t)L[e + 3] * kHid + col];
                                acc = __dadd_rn(acc, (double)x0);
                                acc = __dadd_rn(acc, (double)x1);
                                acc = __dadd_rn(acc, (double)x2);
                                acc = __dadd_rn(acc, (double)x3);
                            }
                            for (; e < n; ++e) acc = __dadd_rn(acc, (double)p.W.W1f[(size_t)L[e] * kHid + col]);
                            float h = (float)acc;
                            h = h > 0.0f ? h : 0.0f;
                            __half hi, lo;
                            split_h(h, hi, lo, ovf);
                            const uint32_t off = kmaj_off(m, col);
                            *reinterpret_cast<__half*>(A_hi + off) = hi;
                            *reinterpret_cast<__half*>(A_lo + off) = lo;
                        }
                    }
                    // ---- broadcast this CTA's h1 slice (core columns 4r..4r+3, rows [0, 8g)) to the cluster
                    const int g8 = (maxrow + 7) >> 3;
                    fence_async_smem();
                    __syncthreads();
                    if (tid == 0) {
                        const uint32_t bytes = (uint32_t)g8 * 128u;
                        for (uint32_t d = 0; d < (uint32_t)kClusterN; ++d) {
                            if (d == rank) continue;
                            const uint32_t cb = map_to(bar_h1, d);
                            mbar_remote_expect_tx(cb, 8u * bytes);
                            for (int sp = 0; sp < 2; ++sp)
                                for (int cc = 0; cc < 4; ++cc) {
                                    const uint32_t off = (uint32_t)sp * kSplitA + (uint32_t)(4 * rank + cc) * kCoreCol;
                                    bulk_s2peer(map_to(smem_u32(A_hi + off), d), smem_u32(A_hi + off), bytes, cb);
                                }
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    mbar_wait_cluster(bar_h1, ph_h1);
                    ph_h1 ^= 1u;
                    // ---- L2 on tcgen05: D1 (cols 0-31), D2 (cols 32-63)
                    tc_fence_before();
                    __syncthreads();
                    tc_fence_after();
                    if (tid == 0) {
                        const uint32_t idesc = idesc_f16(kTileRows, kSliceN);
                        const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo), wb = smem_u32(sm + kOffW2);
                        for (int ks = 0; ks < kHid / 16; ++ks) {
                            const uint64_t dah = umma_desc(ah + (uint32_t)ks * 2u * kCoreCol, kCoreCol, 128);
                            const uint64_t dal = umma_desc(al + (uint32_t)ks * 2u * kCoreCol, kCoreCol, 128);
                            const uint64_t dbh = umma_desc(wb + (uint32_t)ks * 2u * kW2Split, (kSliceN / 8) * 128, 128);
                            const uint64_t dbl = umma_desc(wb + (uint32_t)ks * 2u * kW2Split + kW2Split, (kSliceN / 8) * 128, 128);
                            umma_f16(tmem + 0, dah, dbh, idesc, ks > 0 ? 1u : 0u);
                            umma_f16(tmem + 32, dah, dbl, idesc, ks > 0 ? 1u : 0u);
                            umma_f16(tmem + 32, dal, dbh, idesc, 1u);
                        }
                        umma_commit(bar_mma);
                    }
                    mbar_wait(bar_mma, ph_mma);
                    ph_mma ^= 1u;
                    tc_fence_after();
                    // ---- E2: h2 slice -> H2 (fp16 split, K = 32)
                    {
                        const int q4 = warp & 3, hc = warp >> 2;
                        const bool any = (n_s[2 * q4] > 0) || (n_s[2 * q4 + 1] > 0);
                        if (any) {
                            uint32_t d1[16], d2[16];
                            const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
                            tmem_ld16(tl + (uint32_t)(16 * hc), d1);
                            tmem_ld16(tl + (uint32_t)(32 + 16 * hc), d2);
                            tmem_wait_ld();
                            const int m = 32 * q4 + lane;
                            const float inv = 1.0f / kLo;
#pragma unroll
                            for (int g = 0; g < 2; ++g) {
                                __half hi[8], lo[8];
#pragma unroll
                                for (int t = 0; t < 8; ++t) {
                                    const int cl = 16 * hc + 8 * g + t;
                                    float z = __fmaf_rn(__uint_as_float(d2[8 * g + t]), inv, __uint_as_float(d1[8 * g + t]));
                                    z = __fmaf_rn(z, p.W.s2u, b2s[cl]);
                                    z = z > 0.0f ? z : 0.0f;
                                    split_h(z, hi[t], lo[t], ovf);
                                }
                                const uint32_t off = kmaj_off(m, 16 * hc + 8 * g);
                                *reinterpret_cast<uint4*>(H2_hi + off) = make_uint4(pack_half2(hi[0], hi[1]), pack_half2(hi[2], hi[3]), pack_half2(hi[4], hi[5]), pack_half2(hi[6], hi[7]));
                                *reinterpret_cast<uint4*>(H2_lo + off) = make_uint4(pack_half2(lo[0], lo[1]), pack_half2(lo[2], lo[3]), pack_half2(lo[4], lo[5]), pack_half2(lo[6], lo[7]));
                            }
                        }
                    }
                    fence_async_smem();
                    tc_fence_before();
                    __syncthreads();
                    tc_fence_after();
                    // ---- L3 on tcgen05: partial outputs of this CTA's 32 h2 columns, Da (64-79), Db (80-95)
                    if (tid == 0) {
                        const uint32_t idesc = idesc_f16(kTileRows, 16);
                        const uint32_t hh = smem_u32(H2_hi), hl = smem_u32(H2_lo), w3 = smem_u32(sm + kOffW3);
                        for (int ks = 0; ks < kSliceN / 16; ++ks) {
                            const uint64_t dah = umma_desc(hh + (uint32_t)ks * 2u * kCoreCol, kCoreCol, 128);
                            const uint64_t dal = umma_desc(hl + (uint32_t)ks * 2u * kCoreCol, kCoreCol, 128);
                            const uint64_t dbh = umma_desc(w3 + (uint32_t)ks * 2u * kW3Split, (16 / 8) * 128, 128);
                            const uint64_t dbl = umma_desc(w3 + (uint32_t)ks * 2u * kW3Split + kW3Split, (16 / 8) * 128, 128);
                            umma_f16(tmem + 64, dah, dbh, idesc, ks > 0 ? 1u : 0u);
                            umma_f16(tmem + 80, dah, dbl, idesc, ks > 0 ? 1u : 0u);
                            umma_f16(tmem + 80, dal, dbh, idesc, 1u);
                        }
                        umma_commit(bar_mma);
                    }
                    mbar_wait(bar_mma, ph_mma);
                    ph_mma ^= 1u;
                    tc_fence_after();
                    if (warp < 4) {
                        const int q4 = warp;
                        const bool any = (n_s[2 * q4] > 0) || (n_s[2 * q4 + 1] > 0);
                        if (any) {
                            uint32_t da[8], db[8];
                            const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
                            tmem_ld8(tl + 64u, da);
                            tmem_ld8(tl + 80u, db);
                            tmem_wait_ld();
                            const int m = 32 * q4 + lane;
                            double pv[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                pv[k] = __dadd_rn((double)__uint_as_float(da[k]), (double)__uint_as_float(db[k]) * (1.0 / 2048.0));
                            double2* dst = reinterpret_cast<double2*>(part_out + m * 8);
                            dst[0] = make_double2(pv[0], pv[1]);
                            dst[1] = make_double2(pv[2], pv[3]);
                            dst[2] = make_double2(pv[4], pv[5]);
                            dst[3] = make_double2(pv[6], pv[7]);
                        }
                    }
                    // ---- partials of row block s -> CTA s
                    fence_async_smem();
                    tc_fence_before();
                    __syncthreads();
                    if (tid == 0) {
                        for (uint32_t s = 0; s < (uint32_t)kClusterN; ++s) {
                            const uint32_t bytes = (uint32_t)n_s[s] * 64u;
                            const uint32_t cb = map_to(bar_part, s);
                            mbar_remote_expect_tx(cb, bytes);
                            if (bytes)
                                bulk_s2peer(map_to(smem_u32(part_in + rank * kRoundRows * 8), s),
                                            smem_u32(part_out + s * kRoundRows * 8), bytes, cb);
                        }
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    mbar_wait_cluster(bar_part, ph_part);
                    ph_part ^= 1u;
                    // ---- E3 for this CTA's own rows: thread (row i, hop k)
                    if (tid < kRoundRows * 8) {
                        const int i = tid >> 3, k = tid & 7;
                        const bool valid = i < own_n;
                        double Gk = 0.0, Ek = 0.0;
                        if (valid) {
                            double acc = 0.0;
#pragma unroll
                            for (int s = 0; s < kClusterN; ++s) acc = __dadd_rn(acc, part_in[(s * kRoundRows + i) * 8 + k]);
                            const double out = __dadd_rn(b3s[k], __dmul_rn(acc, p.W.s3u));
                            Ek = out > 0.0 ? out : 0.0;
                            const uint8_t wk = wreq[i * kWin + k];
                            Gk = (wk != (uint8_t)kVac) ? arrhenius(Ek, p.P) : 0.0;
                        }
                        double R = 0.0;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) R = __dadd_rn(R, __shfl_sync(0xffffffffu, Gk, (lane & ~7) + kk));
                        if (valid) {
                            if (phase_mode) {
                                const int r = c.miss[kRoundRows * k_round + i];
                                rowG[r * 8 + k] = Gk;
                                MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                                me[0].G[k] = Gk;
                                if (k == 0) { rowR[r] = R; rowC[r] = 0; me[0].R = R; me[0].clamps = 0; }
                            } else {
                                const int g = c.ebase + i;
                                const int slot = p.windows ? g : (p.rows ? p.rows[g] : g);
                                if (p.rates) p.rates[(size_t)slot * 8 + k] = Gk;
                                if (p.E) p.E[(size_t)slot * 8 + k] = Ek;
                                if (k == 0 && p.Rsum) p.Rsum[slot] = R;
                            }
                        }
                    }
                }
                if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncthreads();
                ++k_round;
                if (!any_more) break;
            }
            if (all_dead) break;
            if (!phase_mode) continue;
        }

        // ================= BKL step per running domain (thread per domain) =================
        __syncthreads();
        if (tid < c.nseg && c.seg_run[tid]) {
            const int i = tid;
            const int cnt = c.seg_cnt[i], moff = c.seg_moff[i];
            double lbuf[32];
            int lidx[16];
            const bool small = cnt <= 16;
            double* buf = small ? lbuf : p.scratch + 4 * (size_t)c.seg_goff[i];
            int* idx = small ? lidx : p.iscratch + c.seg_goff[i];
            int m = 0;
            unsigned long long cl = 0;
            for (int a = 0; a < cnt; ++a)
                if (c.mem_act[moff + a]) {
                    const int r = c.mem_row[moff + a];
                    buf[m] = rowR[r];
                    cl += (unsigned long long)rowC[r];
                    idx[m] = a;
                    ++m;
                }
            bool stop = false;
            if (m == 0) {
                stop = true;
            } else {
                atomicAdd(&c.evals, 8ull * (unsigned long long)m);
                if (cl) atomicAdd(&c.clamps, cl);
                int P = 1, nlev = 0;
                const double Rd = tree_build(buf, m, P, nlev);
                if (!(Rd > 0.0)) {
                    stop = true;
                } else {
                    const unsigned long long ph = (unsigned long long)p.ph->phase;
                    double u_sel, u_t;
                    philox_uniforms(p.S.seed, make_uint4(c.seg_it[i], (uint32_t)c.seg_dom[i], (uint32_t)ph, (uint32_t)(ph >> 32)),
                                    u_sel, u_t);
                    const double dt = __ddiv_rn(-det_log(u_t), Rd);
                    if (__dadd_rn(c.seg_t[i], dt) > p.S.window) {
                        stop = true;                          // overshooting draw discarded
                    } else {
                        double rr = __dmul_rn(u_sel, Rd);
                        const int leaf = tree_descend(buf, m, P, nlev, rr);
                        const int a = idx[leaf];
                        const int slot = c.mem_slot[moff + a];
                        const int k = pick_hop(rowG + (size_t)c.mem_row[moff + a] * 8, rr);
                        const int4 ov = c.mem_vac[moff + a];
                        const int4 nv = apply_hop(p.species, p.vac, slot, k, p.F, p.G);
                        c.mem_vac[moff + a] = nv;
                        long long d2;
                        int sec2;
                        dom_sector(nv, p.S, d2, sec2);
                        if (d2 != c.seg_dom[i] || sec2 != p.ph->sector) c.mem_act[moff + a] = 0;
                        if (p.S.log) {
                            if (near_face(p.F, ov.y, ov.z, ov.w))
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, ov.y, ov.z, ov.w,
                                          p.species[site_of(p.F, ov.x, ov.y, ov.z, ov.w)]);
                            if (near_face(p.F, nv.y, nv.z, nv.w))
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, nv.y, nv.z, nv.w, kVac);
                            bool out = false;
                            const int np[3] = {nv.y, nv.z, nv.w};
                            for (int ax = 0; ax < 3; ++ax)
                                if (!p.F.wrap[ax] && (np[ax] < 0 || np[ax] >= 2 * p.F.L[ax])) out = true;
                            if (out) {
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, nv.y, nv.z, nv.w, kMigrateBase + p.S.gid[slot]);
                                p.vac[slot].x = -1;
                            }
                        }
                        c.seg_t[i] = __dadd_rn(c.seg_t[i], dt);
                        c.seg_it[i] += 1u;
                        atomicAdd(&c.events, 1ull);
                    }
                }
            }
            if (stop) c.seg_run[i] = 0;
        }
        __syncthreads();
        if (tid == 0) {
            int nr = 0;
            for (int i = 0; i < c.nseg; ++i) nr += c.seg_run[i];
            c.nrun = nr;
        }
    }

    // ---- teardown
    if (ovf && p.overflow) atomicAdd(p.overflow, ovf);
    __syncthreads();
    if (tid == 0 && phase_mode) {
        if (c.events) atomicAdd(&p.ctr->events, c.events);
        if (c.evals) atomicAdd(&p.ctr->hop_evals, c.evals);
        if (c.clamps) atomicAdd(&p.ctr->clamps, c.clamps);
        if (c.mrows) atomicAdd(&p.ctr->mrows, c.mrows);
    }
    if (kTC) {
        tc_fence_before();
        cluster_sync();
        if (warp == 2) {
            tc_fence_after();
            tmem_dealloc(tmem, 128);
        }
    }
}

} // namespace

size_t engine_smem_bytes() { return kSmemTotal; }

cudaError_t engine_setup()
{
    cudaError_t e = cudaFuncSetAttribute(engine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTotal);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(engine_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTotal);
}

int engine_max_clusters()
{
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterN;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kClusterN * 64, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemTotal;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, engine_kernel<true>, &cfg) != cudaSuccess) return 0;
    return n;
}

cudaError_t launch_engine(const EngineParams& p, bool tc, int nclusters, int num_sms, cudaStream_t s)
{
    if (!tc) {
        engine_kernel<false><<<num_sms, kThreads, kSmemTotal, s>>>(p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterN;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kClusterN * nclusters, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemTotal;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, engine_kernel<true>, p);
}

} // namespace akmc
