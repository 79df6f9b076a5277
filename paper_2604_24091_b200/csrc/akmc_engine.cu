// akmc_engine.cu -- sublattice phase engine (see akmc_engine.cuh) and its barrier-network evaluator.
//
// Control (every CTA, independently): hold up to 32 domains (segments) of the current phase in slots;
// per iteration gather the 64-site window of every active vacancy, look the window up in
// the per-vacancy memo, evaluate the misses, then run one BKL step per running domain (tree over the
// domain's rates, Philox draw, window test, hop) exactly as the oracle's run_sublattice does.  Stopped
// domains free their slots, which are refilled from the phase's segment list (domains of a phase are
// independent, so the processing order does not change any trajectory).
//
// Evaluator, FP32-equivalent mode (cluster of 4 CTAs, rounds in lockstep; tile M = 128 = 4 x 32 rows):
//   L1 (CUDA cores, requesting CTA): h1 = ReLU(b1' + sum over the row's non-Fe slots of W1'(s, slot)) --
//      the one-hot layer is a sparse gather-sum (~6 rows of W1'), not a dense contraction -- summed in
//      FP64 in slot order, rounded once to FP32, split into fp16 hi + lo*2^-11 and written to rows
//      [32r, 32r+32) of the A operand; the request multicasts those rows into the other 3 CTAs' A;
//   L2 (tcgen05, M=128 N=64 K=256): CTA r computes columns [64r, 64r+64) with its resident W2 slice:
//      D1 = Ahi*W2hi, D2 = Ahi*W2lo + Alo*W2hi; h2 = ReLU(2^-s2 (D1 + 2^-11 D2) + b2) -> fp16 split;
//   L3 (tcgen05, M=128 N=16 K=64): CTA r's partial of the 8 outputs over its 64 h2 columns; the
//      partials of row block [32s, 32s+32) are bulk-copied to CTA s, which sums them in fixed order
//      (FP64), adds b3, clamps at 0 and forms Gamma = nu0 det_exp(-E/kT).
// The result of a row depends only on its window (rows of a tile do not interact, the order of every
// sum is fixed), so memoisation and any tiling or decomposition give bit-identical trajectories.
// FP64 verify mode: each CTA evaluates its own misses (pair KRA or FP64 MLP, same arithmetic as the
// FP64 kernels), no cluster.
#include "akmc_engine.cuh"
#include "akmc_ptx.cuh"
#include "akmc_eval.cuh"

// Compile-time variants (A/B builds via build.build(out=..., defines=...) and AKMC_LIB; tools/ab_probe.py).
// Defaults are the measured best on B200 (C5, same box, profiles/r01_engine_timing.md):
#ifndef AKMC_REFILL_FAST
#define AKMC_REFILL_FAST 1      // skip slot placement when nothing is pending (-2 %)
#endif
#ifndef AKMC_GATHER_ROWS
#define AKMC_GATHER_ROWS 8      // gather rows per warp in flight (A/B at round-2 HEAD: 12 -> same, 16 -> +8 %)
#endif
#ifndef AKMC_PREFETCH
#define AKMC_PREFETCH 0         // L2 prefetch of the next window/memo at hop/placement (+1.6 %, slower)
#endif
#ifndef AKMC_XCHG_DSMEM
#define AKMC_XCHG_DSMEM 0       // h1 rows by DSMEM bulk copies instead of L2-staged multicast (+5 %, slower)
#endif
#ifndef AKMC_CHAIN_MAX
#define AKMC_CHAIN_MAX 0        // memo-hit chain: extra BKL steps a single-member domain may take per iteration
#endif                          // (bit-exact; C5: 30 % of checks hit, -0.7 iterations/CTA, but 1.86 -> 2.51 ms
#ifndef AKMC_CHAIN_NRUN         //  per sweep with 64; gated to the tail (<= 4 / 16 running domains) 1.97 / 2.04)
#define AKMC_CHAIN_NRUN 1024    // ... only while the CTA holds at most this many running domains
#endif
#ifndef AKMC_ENGINE_L1_ROWS
#define AKMC_ENGINE_L1_ROWS 2   // layer-1 rows per warp call in the engine, W1' rows per row in flight (A/B: 4 x 1,
#endif                          // no spills, 2.05 vs 1.97 ms per C5 sweep)
#ifndef AKMC_ENGINE_L1_BATCH
#define AKMC_ENGINE_L1_BATCH 2
#endif
#ifndef AKMC_PDL
#define AKMC_PDL 1              // programmatic dependent launch of the engine (A/B knob)
#endif
#ifndef AKMC_SERIAL_CLOCK
#define AKMC_SERIAL_CLOCK 1     // serial mode: voxel clock cached in the slot (no per-event global load)
#endif
#ifndef AKMC_L1_PROBE
#define AKMC_L1_PROBE 0         // cycle laps inside layer 1 (diagnostic)
#endif

namespace akmc {

namespace {
constexpr int kEL1Rows = AKMC_ENGINE_L1_ROWS, kEL1Batch = AKMC_ENGINE_L1_BATCH;
using namespace ptx;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileRows = kRoundRows * kClusterN;              // 128
constexpr uint32_t kSplitA = kTileRows * kHid * 2;             // 64 KiB: one fp16 split of h1
constexpr uint32_t kW2Split = kSliceN * 16 * 2;                // 1 KiB: one split of a W2-slice K-step
constexpr uint32_t kW2Bytes = (kHid / 16) * 2 * kW2Split;      // 32 KiB
constexpr uint32_t kW3Bytes = kSliceN * 8 * 8;                // 4 KiB: FP64 W3 rows of this CTA's h2 slice

struct ReqHdr { int n, more, alive, pad; };

constexpr int kMaskWords = (kSlots + 31) / 32;

struct Ctl {
    unsigned seg_dom[kSlots];       // domain ids are < 2^32 (checked at init)
    double seg_t[kSlots];
    int seg_goff[kSlots];           // global member offset (scratch of big trees)
    int seg_cnt[kSlots];
    unsigned seg_it[kSlots];
    uint8_t seg_used[kSlots];       // 0 free, 1 head of a held domain, 2 continuation slot
    uint8_t seg_head[kSlots];       // head slot of a continuation slot
    uint8_t seg_run[kSlots];
    uint8_t seg_new[kSlots];
    unsigned cand_dom[2 * kSlots];  // domains waiting for slots: [0, npend) carried over, then fetched
    int cand_off[2 * kSlots];
    int cand_cnt[2 * kSlots];
    short cand_slot[2 * kSlots];    // placement: slot, or -1 (single-slot, parallel) / -2 (deferred)
    int nmulti_def, nfree_single;
    unsigned frees[kMaskWords];     // free slots left for single-slot domains, and their prefix counts
    int fpre[kMaskWords + 1];
    int npend, nnew, fetch, drained, ntot, s0, nhot;
    int int_drained, bready, bdrained, ntot2;   // multi-rank overlap: interior list exhausted; boundary list
                                                 // published, exhausted, size
    unsigned long long bwait0;        // globaltimer when this CTA started waiting for the boundary list
    unsigned freew[kMaskWords], runw[kMaskWords];
    int nrows, nmiss, nrun, ebase;
    int wsum[kWarps];
    int4 mem_vac[kRowCap];          // positions of the held vacancies (this CTA is their only writer)
    int mem_slot[kRowCap];
    short mem_row[kRowCap];
    short row_mem[kRowCap];
    short miss[kRowCap];
    uint8_t mem_act[kRowCap];
    uint8_t mem_seg[kRowCap];       // head slot of the member's domain
    uint8_t row_hit[kRowCap];
    uint8_t row_way[kRowCap];       // memo way that holds the row's current rates (read by the selection)
    unsigned long long events, evals, mrows, clamps;
    // dataflow sweep (p.df): phase (0..7) and my-tile index of each slot / candidate; my tiles' progress
    uint8_t seg_q[kSlots], seg_tp[kSlots];
    uint8_t cand_q[2 * kSlots], cand_tp[2 * kSlots];
    int df_tile[kMyTiles];
    int df_left[kMyTiles];          // domains of the tile's current phase still running
    uint8_t df_np[kMyTiles];        // next phase to activate (8 = sweep done for this tile)
    uint8_t df_ready[kMyTiles];
    uint8_t df_cand[kMyTiles];
    int df_ntiles, df_done_all, df_ring_head, df_nready;
};
constexpr int kDfCand = 16;         // dataflow: tiles tested for readiness per refill

// shared-memory carve-up (offsets from a 1024-aligned base)
constexpr uint32_t kOffA = 0;                                        // h1 hi [0,64K) lo [64K,128K); FP64 scratch
constexpr uint32_t kOffW2 = kOffA + 2 * kSplitA;
constexpr uint32_t kOffW3 = kOffW2 + kW2Bytes;
constexpr uint32_t kOffHdr = kOffW3 + kW3Bytes;                      // [8 sources] ReqHdr
constexpr uint32_t kOffPart = kOffHdr + kClusterN * 16;              // [8 sources][16 rows][8] double
constexpr uint32_t kOffWin = kOffPart + kClusterN * kRoundRows * 8 * 8;   // rows' 1NN window bytes [kRowCap][8]
constexpr uint32_t kOffRowR = kOffWin + kRowCap * 8;                 // [kRowCap] double (a row's 8 rates stay in the memo)
constexpr uint32_t kOffRowC = kOffA + 16384;                         // [kRowCap] int, FP64 mode only (A is scratch there)
constexpr uint32_t kOffB2 = kOffRowR + kRowCap * 8;                  // float [kSliceN]
constexpr uint32_t kOffB3 = kOffB2 + kSliceN * 4;                    // double [8]
constexpr uint32_t kOffL1N = kOffB3 + 8 * 8;                         // [kRowCap] uint8 non-Fe slot count
constexpr uint32_t kOffL1L = kOffL1N + kRowCap;                      // [kRowCap][kL1List] uint16 W1' row index
constexpr uint32_t kOffCtl = (kOffL1L + kRowCap * kL1List * 2 + 15u) & ~15u;
constexpr uint32_t kOffBar = (kOffCtl + (uint32_t)sizeof(Ctl) + 7u) & ~7u;
constexpr int kNumBars = 4;                                          // req, part, mma, weights
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemUsed = kOffTmem + 16;
constexpr uint32_t kSmemTotal = kSmemUsed + 128;                     // 128-B alignment slack (no-swizzle layouts)
template <int N> struct SmemIs; static_assert(kSmemTotal <= 232448, "shared memory budget");
#ifdef AKMC_PRINT_SMEM
SmemIs<kSmemTotal> smem_is;
SmemIs<(int)sizeof(Ctl)> ctl_is;
#endif
static_assert(kTileRows * 8 * 8 <= (kRoundRows / 8) * kRowGroupA,
              "layer-3 partials (and the pair scratch) fit in the CTA's own row block of A (hi / lo)");
static_assert(kOffHdr % 16 == 0 && kOffPart % 16 == 0 && kOffW2 % 16 == 0 && kOffW3 % 16 == 0, "bulk alignment");
static_assert(kRowCap <= 256, "row scan covers one element per thread");
static_assert(kSlots <= kThreads && 2 * kSlots <= kThreads, "slot and candidate threads fit the CTA");


// exclusive block prefix of v over threads [0, 256); total gets the sum (all threads)
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
    for (int w = 0; w < kWarps; ++w) {
        const int t = wsum[w];
        if (w < wid) base += t;
        total += t;
    }
    return base + incl - v;
}



// does TMEM lane quadrant q (tile rows [32q, 32q+32)) hold any valid row of this round?
__device__ __forceinline__ bool quad_has_rows(const int (&n_s)[kClusterN], int q)
{
    bool any = false;
#pragma unroll
    for (int s = 0; s < kClusterN; ++s)
        if (n_s[s] > 0 && s * kRoundRows < 32 * q + 32 && s * kRoundRows + n_s[s] > 32 * q) any = true;
    return any;
}


// layer 1 of up to two rows, all 256 columns (lane = columns 8*lane .. 8*lane+7): FP64 sum of b1' and the
// W1' rows of the window's non-Fe slots in slot order, one rounding to FP32, ReLU, fp16 hi/lo split into
// row m of the A operand (M-major no-swizzle: 8-row group g at g*4096, core column c at c*128) and into the
// CTA's L2 staging block.  The two rows' loads are interleaved (independent latency chains).
// L2 prefetch of what the next gather of a vacancy reads: the <= 8 bricks its window touches (reach 2 cells)
// and its two memo ways
__device__ __forceinline__ void prefetch_l2(const void* ptr) { asm volatile("prefetch.global.L2 [%0];" :: "l"(ptr)); }
__device__ __forceinline__ void prefetch_vacancy(const uint8_t* species, const Frame& F, const int4& v, const void* memo2)
{
    // (clamped to the storage: a vacancy that just left a decomposed block may sit half a cell outside it)
    const int pv[3] = {v.y, v.z, v.w};
    int b0[3], b1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b0[a] = max(0, (((pv[a] - 4) >> 1) + kHalo) >> 2);
        b1[a] = min(F.NB[a] - 1, (((pv[a] + 4) >> 1) + kHalo) >> 2);
    }
    const uint8_t* vb = species + (int64_t)v.x * F.sites;
    for (int bz = b0[2]; bz <= b1[2]; ++bz)
        for (int by = b0[1]; by <= b1[1]; ++by)
            for (int bx = b0[0]; bx <= b1[0]; ++bx)
                prefetch_l2(vb + ((int64_t)((uint32_t)bx + (uint32_t)F.NB[0] * ((uint32_t)by + (uint32_t)F.NB[1] * (uint32_t)bz)) << 7));
    const uint8_t* m = reinterpret_cast<const uint8_t*>(memo2);
    prefetch_l2(m); prefetch_l2(m + 128); prefetch_l2(m + 256);
}

// ---------------------------------------------------------------- dataflow sweep helpers (f1)
// The synchronous sweep (reading A19) runs phase q of every domain after phase q-1 of every domain.  Domain (d, q)
// reads the lattice within 2.5 cells of its sector and writes within 0.5 cell; both lie inside d and its 26
// neighbour domains, and a domain's phase-q sector is >= 3 cells from any other domain's phase-q sector (A20).
// So (d, q) sees exactly the synchronous state as soon as d and its 26 neighbours have finished phase q-1, and it
// can disturb nothing a neighbour still has to read in phase q-1 (they are done).  Tiles of tdom^3 domains carry
// that readiness (a tile's 27 neighbour tiles contain every neighbour of its domains): tile T starts phase q once
// the 27 tiles around it have published done_phase >= q-1 -- the paper's per-sublattice readiness signals
// (P:405-418), here between tiles of one GPU.  Trajectories are those of the synchronous sweep, bit for bit.
__device__ __forceinline__ long long ld_acquire_gpu_s64(const long long* ptr)
{
    long long v;
    asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(ptr) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_s64(long long* ptr, long long v)
{
    asm volatile("st.release.gpu.global.s64 [%0], %1;" :: "l"(ptr), "l"(v) : "memory");
}
__device__ __forceinline__ int df_tile_of(const EngineParams& p, long long d)
{
    const long long v = d / p.S.ndom_vox;
    long long r = d - v * p.S.ndom_vox;
    const int dx = (int)(r % p.S.ND[0]);
    r /= p.S.ND[0];
    const int dy = (int)(r % p.S.ND[1]), dz = (int)(r / p.S.ND[1]);
    const int ntv = p.NT[0] * p.NT[1] * p.NT[2];
    return (int)v * ntv + dx / p.tdom[0] + p.NT[0] * (dy / p.tdom[1] + p.NT[1] * (dz / p.tdom[2]));
}
__device__ __forceinline__ int df_neighbour(const EngineParams& p, int T, int n)
{
    const int ntv = p.NT[0] * p.NT[1] * p.NT[2];
    const int v = T / ntv, r = T - v * ntv;
    int t[3] = {r % p.NT[0], (r / p.NT[0]) % p.NT[1], r / (p.NT[0] * p.NT[1])};
    const int dd[3] = {n % 3 - 1, (n / 3) % 3 - 1, n / 9 - 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) t[a] = (t[a] + dd[a] + p.NT[a]) % p.NT[a];
    return v * ntv + t[0] + p.NT[0] * (t[1] + p.NT[1] * t[2]);
}
// warp bitonic sort of up to 64 keys (2 per lane: lane l holds keys l and l + 32), ascending
__device__ __forceinline__ void warp_sort64(unsigned long long& a, unsigned long long& b)
{
    const int lane = threadIdx.x & 31;
    // element index e: a -> lane, b -> lane + 32
    for (int k = 2; k <= 64; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                // partners are a <-> b of the same lane
                const bool up = ((lane & k) == 0);
                const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
                a = up ? lo : hi; b = up ? hi : lo;
            } else {
                const unsigned long long pa = __shfl_xor_sync(0xffffffffu, a, j);
                const unsigned long long pb = __shfl_xor_sync(0xffffffffu, b, j);
                const bool lower = (lane & j) == 0;
                const bool upa = ((lane & k) == 0), upb = (((lane + 32) & k) == 0);
                a = (lower == upa) ? (a < pa ? a : pa) : (a < pa ? pa : a);
                b = (lower == upb) ? (b < pb ? b : pb) : (b < pb ? pb : b);
            }
        }
    }
}

// the general (slow) activation: any number of vacancies in the set; keys sorted in the ring by lane 0
__device__ __noinline__ void df_activate_slow(const EngineParams& p, Ctl& c, int i)
{
    const int lane = threadIdx.x & 31;
    {
    const int T = c.df_tile[i], q = c.df_np[i];
    const int sector = p.ph[q].sector;
    const long long phase = p.ph[q].phase;
    const int b0 = p.tile_off[T], nb = p.tile_off[T + 1] - b0;
    const int na = min(*(volatile int*)(p.arr_cnt + T), kArrCap);
    // pass 1: count the vacancies now in (tile T, sector of phase q)
    auto keep = [&](int e, int& slot, long long& d) -> bool {
        slot = e < nb ? p.tile_mem[b0 + e] : *(volatile int*)(p.arr_slot + (size_t)T * kArrCap + (e - nb));
        if (slot < 0) return false;
        const int4 v = __ldcv(p.vac + slot);
        if (v.x < 0) return false;
        int sec = 0;
        dom_sector(v, p.S, d, sec);
        return sec == sector && df_tile_of(p, d) == T;
    };
    int n = 0;
    for (int e0 = 0; e0 < nb + na; e0 += 32) {
        int slot; long long d;
        const bool k = (e0 + lane < nb + na) && keep(e0 + lane, slot, d);
        n += __popc(__ballot_sync(0xffffffffu, k));
    }
    int r0 = 0;
    if (lane == 0) r0 = atomicAdd(&c.df_ring_head, n);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    const size_t rb = (size_t)blockIdx.x * p.ring_cap;
    bool ok = r0 + n <= p.ring_cap;
    if (!ok && lane == 0) atomicAdd(p.df_err, 1);
    if (ok) {
        // pass 2: keys (domain << 32 | slot) into the ring
        int w = 0;
        for (int e0 = 0; e0 < nb + na; e0 += 32) {
            int slot = 0; long long d = 0;
            const bool k = (e0 + lane < nb + na) && keep(e0 + lane, slot, d);
            const unsigned bm = __ballot_sync(0xffffffffu, k);
            if (k) p.ring_key[rb + r0 + w + __popc(bm & lanemask_lt())] =
                ((unsigned long long)d << 32) | (unsigned long long)(unsigned)slot;
            w += __popc(bm);
        }
        __syncwarp();
        // sort by (domain, slot): the synchronous order of a competing set (A17)
        if (n <= 64) {
            unsigned long long ka = lane < n ? p.ring_key[rb + r0 + lane] : ~0ull;
            unsigned long long kb = lane + 32 < n ? p.ring_key[rb + r0 + lane + 32] : ~0ull;
            warp_sort64(ka, kb);
            if (lane < n) p.ring_key[rb + r0 + lane] = ka;
            if (lane + 32 < n) p.ring_key[rb + r0 + lane + 32] = kb;
        } else if (lane == 0) {
            unsigned long long* kk = p.ring_key + rb + r0;
            for (int x = 1; x < n; ++x) {
                const unsigned long long v = kk[x];
                int y = x - 1;
                while (y >= 0 && kk[y] > v) { kk[y + 1] = kk[y]; --y; }
                kk[y + 1] = v;
            }
        }
        __syncwarp();
        if (lane == 0) {
            // distinct entries (a vacancy can be listed twice: base list and arrivals) -> members,
            // runs of one domain -> candidate segments
            const unsigned long long* kk = p.ring_key + rb + r0;
            int nseg = 0, m = 0;
            unsigned long long prev = ~0ull;
            long long pd = -1;
            for (int x = 0; x < n; ++x) {
                if (kk[x] == prev) continue;
                prev = kk[x];
                const long long d = (long long)(kk[x] >> 32);
                if (d != pd) { ++nseg; pd = d; }
                ++m;
            }
            const int cq = atomicAdd(&c.nnew, nseg);
            if (cq + nseg > 2 * kSlots) {
                atomicSub(&c.nnew, nseg);          // no room: the tile stays ready for a later refill
            } else {
                int sidx = cq - 1, mi = 0;
                prev = ~0ull; pd = -1;
                for (int x = 0; x < n; ++x) {
                    if (kk[x] == prev) continue;
                    prev = kk[x];
                    const long long d = (long long)(kk[x] >> 32);
                    const int slot = (int)(unsigned)(kk[x] & 0xFFFFFFFFull);
                    if (d != pd) {
                        ++sidx; pd = d;
                        c.cand_dom[sidx] = (unsigned)d;
                        c.cand_off[sidx] = (int)(rb + r0 + mi);
                        c.cand_cnt[sidx] = 0;
                        c.cand_q[sidx] = (uint8_t)q;
                        c.cand_tp[sidx] = (uint8_t)i;
                    }
                    p.ring_slot[rb + r0 + mi] = slot;
                    p.ring_pos[rb + r0 + mi] = __ldcv(p.vac + slot);
                    c.cand_cnt[sidx] += 1;
                    ++mi;
                }
                c.df_np[i] = (uint8_t)(q + 1);
                c.df_left[i] = nseg;
                if (nseg == 0) st_release_gpu_s64(p.done_phase + T, phase);   // empty: done at once
            }
        }
    }
                    }
}

// Activation of my tile i for its next phase (one warp): the vacancies now in (tile, sector of that phase) --
// the tile's sweep-start members plus the vacancies that entered it -- sorted by (domain, slot), duplicates
// dropped, one candidate segment per domain (the synchronous phase's competing sets, A17), members and their
// positions into this CTA's ring.  All loads of up to 256 entries in flight at once; sort and segmentation in
// registers (<= 64 entries; a larger set takes df_activate_slow).
__device__ __forceinline__ void df_activate(const EngineParams& p, Ctl& c, int i)
{
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const int T = c.df_tile[i], q = c.df_np[i];
    const int sector = p.ph[q].sector;
    const long long phase = p.ph[q].phase;
    const int b0 = p.tile_off[T], nb = p.tile_off[T + 1] - b0;
    const int na = min(__ldcv(p.arr_cnt + T), kArrCap);
    const int ntot = nb + na;
    unsigned long long ka = ~0ull, kb = ~0ull;
    int n = 0;
    constexpr int kU = 8;
    for (int e0 = 0; e0 < ntot; e0 += 32 * kU) {
        int sl[kU];
        int4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int e = e0 + 32 * u + lane;
            sl[u] = e < nb ? p.tile_mem[b0 + e] : (e < ntot ? __ldcv(p.arr_slot + (size_t)T * kArrCap + (e - nb)) : -1);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = sl[u] >= 0 ? __ldcv(p.vac + sl[u]) : make_int4(-1, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            bool k = false;
            unsigned long long key = 0;
            if (v[u].x >= 0) {
                long long d;
                int sec;
                dom_sector(v[u], p.S, d, sec);
                k = sec == sector && df_tile_of(p, d) == T;
                key = ((unsigned long long)d << 32) | (unsigned long long)(unsigned)sl[u];
            }
            const unsigned m = __ballot_sync(full, k);
            const int ck = __popc(m);
            if (n + ck <= 64) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pos = lane + 32 * h - n;
                    const bool mine = pos >= 0 && pos < ck;
                    const unsigned long long got = __shfl_sync(full, key, mine ? (int)__fns(m, 0, pos + 1) : 0);
                    if (mine) { if (h == 0) ka = got; else kb = got; }
                }
            }
            n += ck;
        }
    }
    if (n > 64) { df_activate_slow(p, c, i); return; }
    warp_sort64(ka, kb);
    const unsigned long long pa = __shfl_up_sync(full, ka, 1), pb0 = __shfl_up_sync(full, kb, 1);
    const unsigned long long a31 = __shfl_sync(full, ka, 31);      // (every lane executes the shuffles)
    const unsigned long long pb = lane == 0 ? a31 : pb0;
    const bool va = lane < n, vb = lane + 32 < n;
    const bool da = va && lane > 0 && ka == pa, db = vb && kb == pb;
    const bool keepa = va && !da, keepb = vb && !db;
    const bool newa = keepa && (lane == 0 || (ka >> 32) != (pa >> 32)), newb = keepb && ((kb >> 32) != (pb >> 32));
    const unsigned lt = lanemask_lt();
    const unsigned ma = __ballot_sync(full, keepa), mb = __ballot_sync(full, keepb);
    const unsigned sa = __ballot_sync(full, newa), sb = __ballot_sync(full, newb);
    const int mtot = __popc(ma) + __popc(mb), nseg = __popc(sa) + __popc(sb);
    int r0 = 0, cq = 0, ok = 1;
    if (lane == 0) {
        r0 = atomicAdd(&c.df_ring_head, mtot);
        if (r0 + mtot > p.ring_cap) { atomicAdd(p.df_err, 1); ok = 0; }
        if (ok) {
            cq = atomicAdd(&c.nnew, nseg);
            if (cq + nseg > 2 * kSlots) { atomicSub(&c.nnew, nseg); ok = 0; }   // no room: stays ready for a later refill
        }
    }
    ok = __shfl_sync(full, ok, 0);
    if (!ok) return;
    r0 = __shfl_sync(full, r0, 0);
    cq = __shfl_sync(full, cq, 0);
    const size_t rb = (size_t)blockIdx.x * p.ring_cap + r0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const bool kp = h ? keepb : keepa, nw = h ? newb : newa;
        const unsigned long long key = h ? kb : ka;
        const int mi = h ? __popc(ma) + __popc(mb & lt) : __popc(ma & lt);
        const int si = h ? __popc(sa) + __popc(sb & lt) : __popc(sa & lt);
        if (kp) {
            const int slot = (int)(unsigned)(key & 0xFFFFFFFFull);
            p.ring_slot[rb + mi] = slot;
            p.ring_pos[rb + mi] = __ldcv(p.vac + slot);
        }
        if (nw) {
            c.cand_dom[cq + si] = (unsigned)(key >> 32);
            c.cand_off[cq + si] = (int)(rb + mi);
            c.cand_q[cq + si] = (uint8_t)q;
            c.cand_tp[cq + si] = (uint8_t)i;
        }
    }
    __syncwarp();
    for (int s2 = lane; s2 < nseg; s2 += 32) {
        const int next = s2 + 1 < nseg ? c.cand_off[cq + s2 + 1] : (int)(rb + mtot);
        c.cand_cnt[cq + s2] = next - c.cand_off[cq + s2];
    }
    __syncwarp();
    if (lane == 0) {
        c.df_np[i] = (uint8_t)(q + 1);
        c.df_left[i] = nseg;
        if (nseg == 0) st_release_gpu_s64(p.done_phase + T, phase);       // empty: done at once
    }
}

template <bool kTC, bool kFast = false, bool kDF = false>
__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ EngineParams p)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    Ctl& c = *reinterpret_cast<Ctl*>(sm + kOffCtl);
    // full 64-byte windows of the held rows live in a per-CTA global scratch (L1/L2-resident); shared memory
    // keeps the 8 first-shell bytes the rates mask and the hop need
    uint8_t* win = p.wstore + (size_t)blockIdx.x * kRowCap * kWin;
    uint8_t* win8 = sm + kOffWin;
    uint8_t* l1n = sm + kOffL1N;
    uint16_t* l1l = reinterpret_cast<uint16_t*>(sm + kOffL1L);
    double* rowR = reinterpret_cast<double*>(sm + kOffRowR);
    int* rowC = reinterpret_cast<int*>(sm + kOffRowC);
    uint8_t* A_hi = sm + kOffA;
    uint8_t* A_lo = sm + kOffA + kSplitA;
    double* part_in = reinterpret_cast<double*>(sm + kOffPart);     // [8][16][8]
    ReqHdr* hdr = reinterpret_cast<ReqHdr*>(sm + kOffHdr);
    float* b2s = reinterpret_cast<float*>(sm + kOffB2);
    double* b3s = reinterpret_cast<double*>(sm + kOffB3);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kOffTmem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr bool fast = kTC && kFast;              // AKMC_PREC_FP16_FAST: hi parts only (no lo MMAs / copies);
                                                     // a separate instantiation, so FP32 mode carries no branch
    const uint32_t rank = kTC ? cluster_rank() : 0u;
    const uint32_t off_lo = pack_off(p.G.off[lane]), off_hi = pack_off(p.G.off[lane + 32]);   // this lane's window slots
    // h2 slice and the layer-3 partials live in this CTA's own row block of A: dead once layer 2 has
    // completed, and no peer ever writes it (peers' multicasts target their own blocks)
    const uint32_t own_block = (uint32_t)(kRoundRows / 8) * rank * kRowGroupA;
    double* part_out = reinterpret_cast<double*>(sm + kOffA + own_block);             // [128][8] S_rank per row
    double* pair_tmp = reinterpret_cast<double*>(sm + kOffA + kSplitA + own_block);    // [128][8] hc = 1 pairs
    const uint32_t bar_req = smem_u32(&bars[0]), bar_part = smem_u32(&bars[1]);
    const uint32_t bar_mma = smem_u32(&bars[2]), bar_w = smem_u32(&bars[3]);
    const bool phase_mode = (p.mode == kEnginePhase);
    const bool mlp = (p.model == 1);
    unsigned long long ovf = 0;
    constexpr uint32_t kStageSplitRows = (uint32_t)(kRoundRows / 8) * kRowGroupA;   // one split of a round's rows
    uint8_t* g_hi = kTC ? p.stage + ((size_t)cluster_id() * kClusterN + rank) * (2u * kStageSplitRows) : nullptr;
    uint8_t* g_lo = kTC ? g_hi + kStageSplitRows : nullptr;

    if (tid == 0 && blockIdx.x == 0 && p.overlap && p.diag) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.ctr->t_e0 = t;
    }
    if (tid == 0) {
        c.npend = 0; c.drained = 0; c.nrun = 0;
        c.int_drained = 0; c.bready = 0; c.bdrained = 0; c.ntot2 = 0; c.bwait0 = 0;
        c.events = 0; c.evals = 0; c.mrows = 0; c.clamps = 0;
        if (kTC) {
            mbar_init(bar_req, kClusterN);
            mbar_init(bar_part, kClusterN);
            mbar_init(bar_mma, 1);
            mbar_init(bar_w, 1);
            mbar_fence_init();
        }
    }
    if (tid < kSlots) { c.seg_used[tid] = 0; c.seg_run[tid] = 0; c.seg_new[tid] = 0; c.seg_head[tid] = 0; c.seg_q[tid] = 0; }
    if (kDF) {
        if (tid < kMyTiles) {
            const int T = (int)blockIdx.x + tid * (int)gridDim.x;
            c.df_tile[tid] = T < p.ntiles ? T : -1;
            c.df_np[tid] = T < p.ntiles ? 0 : 8;
            c.df_left[tid] = 0;
        }
        if (tid == 0) {
            c.df_ntiles = min(kMyTiles, max(0, (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x));
            c.df_done_all = c.df_ntiles == 0;
        }
    }
    if (tid < kRowCap) c.mem_act[tid] = 0;
    uint32_t tmem = 0;
    uint32_t ph_req = 0, ph_part = 0, ph_mma = 0;
    if (kTC) {
        if (warp == 2) tmem_alloc(smem_u32(tmem_slot), 256);
        if (tid < kSliceN) b2s[tid] = p.W.b2[rank * kSliceN + tid];
        if (tid < 8) b3s[tid] = p.W.b3[tid];
        tc_fence_before();
        cluster_sync();                            // every barrier of the cluster initialised
        tc_fence_after();
        tmem = *tmem_slot;
        if (tid == 0) {
            mbar_expect_tx(bar_w, kW2Bytes + kW3Bytes);
            bulk_g2s(smem_u32(sm + kOffW2), p.W.W2img + (size_t)rank * kW2Bytes, kW2Bytes, bar_w);
            bulk_g2s(smem_u32(sm + kOffW3), p.W.W3d + (size_t)rank * kSliceN * 8, kW3Bytes, bar_w);
        }
        mbar_wait(bar_w, 0);
    } else {
        __syncthreads();
    }
    // programmatic dependent launch (AKMC_PDL): everything above -- barriers, TMEM, the weight slices -- overlaps the
    // tail of the kernel this launch depends on; nothing that kernel (or an earlier one) writes is read before here
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) {
        c.ntot = phase_mode ? (p.serial ? p.nseg_host : (int)p.ctr->nseg) : 0;
        c.nhot = (phase_mode && !p.serial && p.seg_cap > 0) ? (int)p.ctr->nhot : -1;
    }
    __syncthreads();
    const int nrows_eval = (!phase_mode) ? (p.nrows_dev ? *p.nrows_dev : p.nrows_host) : 0;
    // diagnostics (thread 0): iterations, rounds, evaluation rounds, cycles in control / rounds / selection
    unsigned long long d_it = 0, d_rounds = 0, d_erounds = 0, d_refill = 0;
    long long d_cc = 0, d_cr = 0, d_cs = 0;
    long long d_x[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // sub-phase cycles: refill, rows, gather | L1, xchg, L2+E2, L3+part, E3
    long long d_y[4] = {0, 0, 0, 0};              // L1 lap split: memo move | layer 1 | async fences + barrier
    long long d_z[4] = {0, 0, 0, 0};              // AKMC_L1_PROBE: layer-1 sub-steps of warp 0
    long long d_xk = 0;                            // exchange wait of rounds k > 0 (no control before them)
    long long d_df[4] = {0, 0, 0, 0};              // dataflow refill: candidates, readiness, activation, placement
    const long long t_start = clock64();
    unsigned long long my_events = 0, my_evals = 0, my_clamps = 0;   // selection counters (slot threads)
    unsigned long long my_chain = 0, my_check = 0;                    // memo-hit chain: events taken, checks
    long long t_mark = t_start;
    auto lap = [&](long long& acc) { const long long t = clock64(); acc += t - t_mark; t_mark = t; };
    // watchdog progress words (thread 0; mapped host memory, read by the host while the kernel runs)
    auto wd = [&](int code, int a, int b) {
        if (p.watch && tid == 0) {
            volatile int* w = p.watch + blockIdx.x * 8;
            w[0] = (int)d_it; w[1] = code; w[2] = a; w[3] = b; w[4] = c.nrun; w[5] = c.drained; w[6] = c.npend;
            w[7] = p.ph ? (int)p.ph->phase : -1;
            __threadfence_system();
        }
    };

    // per-iteration trace (AKMC_PHASE_TIMING): thread 0 snapshots its counters at the top of every iteration
    long long tr_ctl = 0, tr_rd = 0, tr_sel = 0, tr_t0 = 0;
    unsigned long long tr_rounds = 0;
    int tr_it = 0;
    auto trace_begin = [&]() {
        if (p.diag && tid == 0) {
            tr_ctl = d_x[0] + d_x[1] + d_x[2];
            tr_rd = d_y[0] + d_y[1] + d_y[2] + d_x[4] + d_x[5] + d_x[6] + d_x[7] + d_cr;
            tr_sel = d_cs; tr_rounds = d_rounds; tr_t0 = clock64();
        }
    };
    auto trace_end = [&]() {
        if (p.diag && tid == 0 && phase_mode) {
            unsigned long long* t = p.diag + 96 + 8 * (size_t)min(tr_it, 63);
            atomicAdd(t + 0, 1ull);
            atomicAdd(t + 1, (unsigned long long)c.nrows);
            atomicAdd(t + 2, (unsigned long long)c.nmiss);
            atomicAdd(t + 3, (unsigned long long)c.nrun);
            atomicAdd(t + 4, (unsigned long long)(d_x[0] + d_x[1] + d_x[2] - tr_ctl));
            atomicAdd(t + 5, (unsigned long long)(d_y[0] + d_y[1] + d_y[2] + d_x[4] + d_x[5] + d_x[6] + d_x[7] + d_cr - tr_rd));
            atomicAdd(t + 6, (unsigned long long)(d_cs - tr_sel));
            atomicAdd(t + 7, d_rounds - tr_rounds);
            ++tr_it;
        }
    };

    for (;;) {
        int own_alive = 0;
        trace_begin();
        if (phase_mode) {
            // ================= slots: release stopped domains, refill from the segment list =================
            __syncthreads();
            wd(1, 0, 0);
            if (tid < 32 * kMaskWords) {
                // thread = slot; a slot is freed with its domain (head or continuation of a stopped head)
                const int sl = tid;
                const bool real = sl < kSlots;
                const int used = real ? c.seg_used[sl] : 3;
                const int head = used == 2 ? c.seg_head[sl] : sl;
                const bool rel = real && used != 0 && !c.seg_run[head];
                if (rel) {
#pragma unroll
                    for (int a = 0; a < kSlotCap; ++a) c.mem_act[kSlotCap * sl + a] = 0;
                }
                const bool running = real && used == 1 && c.seg_run[sl];
                __syncwarp();
                if (rel) c.seg_used[sl] = 0;
                if (real) c.seg_new[sl] = 0;
                const unsigned fm = __ballot_sync(0xffffffffu, used == 0 || rel);
                const unsigned rm = __ballot_sync(0xffffffffu, running);
                if (lane == 0) { c.freew[warp] = fm; c.runw[warp] = rm; }
            }
            __syncthreads();
            if (tid == 0) {
                int nfree = 0, nrun0 = 0;
#pragma unroll
                for (int w = 0; w < kMaskWords; ++w) { nfree += __popc(c.freew[w]); nrun0 += __popc(c.runw[w]); }
                c.fetch = 0;
                c.nnew = 0;
                // claim at most a fair share of the segment list at a time (few, large domains -- voxels --
                // must not pile up in a handful of CTAs)
                const int share = max(1, (c.ntot + (int)gridDim.x - 1) / (int)gridDim.x);
                const int claim = min(nfree, share);
                if (kDF) {
                    c.fetch = (!c.df_done_all && c.npend == 0 && nfree > 0 && (nfree >= kSlots / 4 || nrun0 == 0)) ? 2 : 0;
                    c.df_ring_head = 0;
                    c.df_nready = 0;
                } else if (!c.drained) {
                    // multi-rank overlap: the boundary domains' list is published (stream-parallel to this launch)
                    // once the previous phase's halo deltas have been applied; it is polled every iteration and
                    // taken before what is left of the interior list (boundary domains start late, so they go first)
                    if (p.overlap && !c.bready) {
                        long long f;
                        asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(f) : "l"(&p.ctr->bready) : "memory");
                        if (f == p.ph[0].phase + 1) {                   // (published as phase + 1: never 0)
                            c.bready = 1;
                            c.ntot2 = (int)*(volatile unsigned long long*)&p.ctr->nseg2;
                        }
                    }
                    if (c.npend == 0 && nfree > 0) {
                        if (p.overlap && c.bready && !c.bdrained) {
                            const int share2 = max(1, (c.ntot2 + (int)gridDim.x - 1) / (int)gridDim.x);
                            const int claim2 = min(nfree, share2);
                            const int s2 = (int)atomicAdd(&p.ctr->chunk2, (unsigned long long)claim2);
                            if (s2 >= c.ntot2) {
                                c.bdrained = 1;
                            } else {
                                c.fetch = 3; c.s0 = s2; c.nnew = min(claim2, c.ntot2 - s2);
                                ++d_refill;
                            }
                        }
                        if (c.fetch == 0 && !c.int_drained && (nfree >= kSlots / 4 || nrun0 == 0)) {
                            const int s0 = (int)atomicAdd(&p.ctr->chunk, (unsigned long long)claim);
                            if (s0 >= c.ntot) {
                                c.int_drained = 1;
                            } else {
                                c.fetch = 1; c.s0 = s0; c.nnew = min(claim, c.ntot - s0);
                                ++d_refill;
                            }
                        }
                    }
                    if (c.int_drained && (!p.overlap || c.bdrained)) {
                        c.drained = 1;
                    } else if (c.int_drained && p.overlap && !c.bready && c.fetch == 0) {
                        // nothing left here but the unpublished boundary list: keep iterating (the cluster peers
                        // are never held up), bounded
                        unsigned long long now;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                        if (!c.bwait0) c.bwait0 = now;
                        if (now - c.bwait0 > 30000000000ull) {          // never published: report, do not hang
                            atomicAdd(p.overflow, 1ull);
                            c.drained = 1;
                        } else if (nrun0 == 0) {
                            __nanosleep(256);
                        }
                    }
                }
            }
            __syncthreads();
            if (kDF && c.fetch == 2) {
                long long tdf = clock64();
                // ---- dataflow activation: which of my tiles may start their next phase, then one tile per warp
                // candidates: tiles whose previous phase is done, lowest next phase first, at most kDfCand per refill
                static_assert(kMyTiles == 32, "one warp ballots over my tiles");
                if (warp == 0) {
                    const int i = lane;
                    const bool el = i < c.df_ntiles && c.df_np[i] < 8 && c.df_left[i] == 0;
                    const int nq = el ? c.df_np[i] : 8;
                    int nc = 0, mine = -1;
                    for (int qq = 0; qq < 8; ++qq) {
                        const unsigned m = __ballot_sync(0xffffffffu, nq == qq);
                        if (nq == qq) mine = nc + __popc(m & lanemask_lt());
                        nc += __popc(m);
                    }
                    const bool take = mine >= 0 && mine < kDfCand;
                    c.df_ready[i] = take ? 1 : 0;
                    if (take) c.df_cand[mine] = (uint8_t)i;
                    if (lane == 0) c.df_nready = min(nc, kDfCand);
                }
                __syncthreads();
                if (tid == 0) { const long long t = clock64(); d_df[0] += t - tdf; tdf = t; }
                // readiness: 27 neighbour tiles' done_phase (relaxed loads, all in flight; one acquire fence after)
                for (int t = tid; t < c.df_nready * 27; t += kThreads) {
                    const int i = c.df_cand[t / 27], n = t % 27;
                    const long long need = p.ph[0].phase + (long long)c.df_np[i] - 1;
                    if (__ldcv(p.done_phase + df_neighbour(p, c.df_tile[i], n)) < need) c.df_ready[i] = 0;
                }
                __threadfence();
                __syncthreads();
                if (tid == 0) { const long long t = clock64(); d_df[1] += t - tdf; tdf = t; }
                {
                    // warp w activates the w-th ready tile
                    int cnt = 0, pick = -1;
                    for (int i = 0; i < c.df_ntiles; ++i)
                        if (c.df_ready[i]) { if (cnt == warp) pick = i; ++cnt; }
                    if (pick >= 0) df_activate(p, c, pick);
                }
                __syncthreads();
                if (tid == 0) { const long long t = clock64(); d_df[2] += t - tdf; tdf = t; }
                if (tid == 0) {
                    int all = 1;
                    for (int i = 0; i < c.df_ntiles; ++i) all &= (c.df_np[i] >= 8) ? 1 : 0;
                    c.df_done_all = all;
                    c.fetch = c.nnew > 0 ? 1 : 0;
                    if (c.fetch) ++d_refill;
                }
            }
            if ((c.fetch == 1 || c.fetch == 3) && !kDF && tid < c.nnew) {
                const int si = c.s0 + tid;
                const Segment sg = c.fetch == 3 ? p.segs2[si]
                                                : p.segs[(c.nhot < 0 || si < c.nhot) ? si : p.seg_cap - 1 - (si - c.nhot)];
                const int q = c.npend + tid;
                c.cand_dom[q] = (unsigned)sg.dom; c.cand_off[q] = sg.off; c.cand_cnt[q] = sg.cnt;
                c.cand_q[q] = 0; c.cand_tp[q] = 0;                        // (one phase per launch: p.ph[0])
            }
            __syncthreads();
            const int ncand = c.npend + c.nnew;     // block-uniform (shared, after a barrier)
#if AKMC_REFILL_FAST
            if (ncand == 0) {                        // nothing to place: running set unchanged
                if (tid == 0) {
                    int nr = 0;
#pragma unroll
                    for (int w = 0; w < kMaskWords; ++w) nr += __popc(c.runw[w]);
                    c.npend = 0;
                    c.nrun = nr;
                }
            } else
#endif
            {
                const bool multi = tid < ncand && c.cand_cnt[tid] > kSlotCap;
                if (tid < ncand) c.cand_slot[tid] = -1;
                const int any_multi = __syncthreads_or(multi ? 1 : 0);
                if (tid == 0) {
    #pragma unroll
                    for (int w = 0; w < kMaskWords; ++w) c.frees[w] = c.freew[w];
                    if (any_multi) {
                        // domains needing several consecutive slots (> 2 vacancies, rare): first fit, sequentially;
                        // single-slot domains are placed in parallel below
                        int nd = 0;
                        for (int q = 0; q < ncand; ++q) {
                            const int cnt = c.cand_cnt[q];
                            if (cnt <= kSlotCap) continue;
                            if (cnt > kRowCap) { atomicAdd(p.overflow, 1ull); c.cand_slot[q] = -3; continue; }
                            const int need = (cnt + kSlotCap - 1) / kSlotCap;
                            int h = -1;
                            for (int i = 0, run = 0; i < kSlots; ++i) {
                                run = ((c.frees[i >> 5] >> (i & 31)) & 1u) ? run + 1 : 0;
                                if (run == need) { h = i - need + 1; break; }
                            }
                            if (h < 0) { c.cand_slot[q] = -2; ++nd; continue; }
                            for (int t = 0; t < need; ++t) c.frees[(h + t) >> 5] &= ~(1u << ((h + t) & 31));
                            c.cand_slot[q] = (short)h;
                            for (int t = 1; t < need; ++t) { c.seg_used[h + t] = 2; c.seg_head[h + t] = (uint8_t)h; }
                        }
                        c.nmulti_def = nd;
                    }
                    c.fpre[0] = 0;
    #pragma unroll
                    for (int w = 0; w < kMaskWords; ++w) c.fpre[w + 1] = c.fpre[w] + __popc(c.frees[w]);
                    c.nfree_single = c.fpre[kMaskWords];
                }
                __syncthreads();
                {
                    // the j-th single-slot candidate takes the j-th free slot; the rest are deferred
                    const bool single = tid < ncand && c.cand_slot[tid] == -1;
                    int nsingle = 0;
                    const int j = block_excl(single ? 1 : 0, c.wsum, nsingle);
                    const int nf = c.nfree_single;
                    if (single) {
                        if (j < nf) {
                            int w = 0;
    #pragma unroll
                            for (int t = 1; t < kMaskWords; ++t)
                                if (c.fpre[t] <= j) w = t;
                            c.cand_slot[tid] = (short)(32 * w + (int)__fns(c.frees[w], 0, j - c.fpre[w] + 1));
                        } else {
                            c.cand_slot[tid] = -2;
                        }
                    }
                    __syncthreads();
                    const int q = tid;
                    const bool deferred = q < ncand && c.cand_slot[q] == -2;
                    int ndef = 0;
                    const int pi = block_excl(deferred ? 1 : 0, c.wsum, ndef);
                    // carried-over domains are compacted in place to the front of the candidate list (read first)
                    unsigned cdom = 0;
                    int coff = 0, ccnt = 0, cslot = -3;
                    uint8_t cq = 0, ctp = 0;
                    if (q < ncand) {
                        cdom = c.cand_dom[q]; coff = c.cand_off[q]; ccnt = c.cand_cnt[q]; cslot = c.cand_slot[q];
                        cq = c.cand_q[q]; ctp = c.cand_tp[q];
                    }
                    __syncthreads();
                    if (deferred) { c.cand_dom[pi] = cdom; c.cand_off[pi] = coff; c.cand_cnt[pi] = ccnt; c.cand_q[pi] = cq; c.cand_tp[pi] = ctp; }
                    if (cslot >= 0) {
                        const int h = cslot;
                        c.seg_q[h] = cq; c.seg_tp[h] = ctp;
                        c.seg_used[h] = 1;
                        c.seg_dom[h] = cdom; c.seg_goff[h] = coff; c.seg_cnt[h] = ccnt;
                        // serial mode: seg_t IS the voxel clock for the launch (same sums as p.clock += dt, no
                        // dependent global load per event); sublattice: the domain's time in the window
                        c.seg_t[h] = (AKMC_SERIAL_CLOCK && p.serial) ? p.clock[cdom] : 0.0;
                        c.seg_it[h] = 0u; c.seg_new[h] = 1;
                        c.seg_run[h] = (p.serial && p.term[cdom]) ? 0 : 1;   // a terminal voxel stays frozen
                    }
                    int nplaced = 0;
                    block_excl(cslot >= 0 ? 1 : 0, c.wsum, nplaced);
                    if (tid == 0) {
                        int nr = 0;
    #pragma unroll
                        for (int w = 0; w < kMaskWords; ++w) nr += __popc(c.runw[w]);
                        c.npend = ndef;
                        c.nrun = nr + nplaced;
                    }
                }
                __syncthreads();
                // members of newly placed domains: slot ids and positions, one member position per thread (all
                // loads in flight at once)
                for (int pm = tid; pm < kRowCap; pm += kThreads) {
                    const int sl = pm / kSlotCap;
                    const int h = c.seg_used[sl] == 2 ? c.seg_head[sl] : sl;
                    const int a = pm - kSlotCap * h;
                    if (c.seg_used[sl] != 0 && c.seg_new[h] && a < c.seg_cnt[h]) {
                        const int goff = c.seg_goff[h];
                        const int slot = p.members[goff + a];
                        const int4 pos = p.serial ? p.vac[slot] : p.mpos[goff + a];
#if AKMC_PREFETCH
                        prefetch_vacancy(p.species, p.F, pos, p.memo + 2 * (size_t)slot);
#endif
                        c.mem_slot[pm] = slot;
                        c.mem_vac[pm] = pos;
                        c.mem_act[pm] = 1;
                        c.mem_seg[pm] = (uint8_t)h;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) lap(d_x[0]);
            own_alive = (c.nrun > 0 || (kDF && (!c.df_done_all || c.npend > 0)) || (p.overlap && !c.drained)) ? 1 : 0;
            // ================= rows = active members of running domains, in slot/member order =================
            int total = 0;
            {
                const bool act = tid < kRowCap && c.mem_act[tid] && c.seg_run[c.mem_seg[tid]];
                const int r = block_excl(act ? 1 : 0, c.wsum, total);
                if (tid < kRowCap) c.mem_row[tid] = act ? (short)r : (short)-1;
                if (act) c.row_mem[r] = (short)tid;
            }
            if (tid == 0) c.nrows = total;
            __syncthreads();
            if (tid == 0) lap(d_x[1]);
            // ================= gather + memo lookup: warp per row, lanes = window slots j and j+32 =================
            const int nrows = c.nrows;
            constexpr int kGR = AKMC_GATHER_ROWS;     // rows per warp in flight
            for (int r0 = warp; r0 < nrows; r0 += kGR * kWarps) {
                // kGR rows per warp in flight: memo ways (lanes 0-15 way 0, 16-31 way 1) and window bytes
                const int k = lane & 15, way = lane >> 4;
                uint32_t kw[kGR];
                double gv[kGR];
                int cv[kGR];
                uint8_t b0[kGR], b1[kGR];
#pragma unroll
                for (int q = 0; q < kGR; ++q) {
                    const int r = r0 + q * kWarps;
                    kw[q] = 0; gv[q] = 0.0; cv[q] = 0; b0[q] = 0; b1[q] = 0;
                    if (r < nrows) {
                        const int pm = c.row_mem[r];
                        const MemoEntry& e = p.memo[2 * (size_t)c.mem_slot[pm] + way];
                        const int4 v = c.mem_vac[pm];
                        kw[q] = reinterpret_cast<const uint32_t*>(e.key)[k];
                        if (k < 8) gv[q] = e.G[k];
                        else if (k == 8) gv[q] = e.R;
                        else if (k == 9) cv[q] = e.clamps;
                        b0[q] = site_byte_pk(p.species, p.F, v, off_lo);
                        b1[q] = site_byte_pk(p.species, p.F, v, off_hi);
                    }
                }
#pragma unroll
                for (int q = 0; q < kGR; ++q) {
                    const int r = r0 + q * kWarps;
                    if (r < nrows) {
                        win[r * kWin + lane] = b0[q];
                        win[r * kWin + lane + 32] = b1[q];
                        if (lane < 8) win8[r * 8 + lane] = b0[q];
                    }
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < kGR; ++q) {
                    const int r = r0 + q * kWarps;
                    if (r >= nrows) break;
                    // window word k (slots 4k..4k+3) assembled from the lanes holding those slots
                    uint32_t ww = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t v0 = __shfl_sync(0xffffffffu, (uint32_t)b0[q], 4 * (k & 7) + j);
                        const uint32_t v1 = __shfl_sync(0xffffffffu, (uint32_t)b1[q], 4 * (k & 7) + j);
                        ww |= (k < 8 ? v0 : v1) << (8 * j);
                    }
                    const unsigned eq = __ballot_sync(0xffffffffu, ww == kw[q]);
                    const int hit = (eq & 0xFFFFu) == 0xFFFFu ? 0 : ((eq >> 16) == 0xFFFFu ? 1 : -1);
                    if (hit >= 0 && way == hit) {
                        if (k == 8) rowR[r] = gv[q];
                        else if (k == 9 && !kTC) rowC[r] = cv[q];
                    }
                    if (lane == 0) { c.row_hit[r] = hit >= 0 ? 1 : 0; c.row_way[r] = hit > 0 ? 1 : 0; }
                    if (kTC && hit < 0) l1_list_store(r, b0[q], b1[q], l1n, l1l);
                }
            }
            __syncthreads();
            {
                const bool ms = tid < nrows && !c.row_hit[tid];
                const int q = block_excl(ms ? 1 : 0, c.wsum, total);
                if (ms) c.miss[q] = (short)tid;
            }
            if (tid == 0) { c.nmiss = total; c.mrows += (unsigned long long)total; }
            __syncthreads();
            wd(3, c.nrows, c.nmiss);
        }
        if (tid == 0) { lap(d_x[2]); ++d_it; }

        // ================= evaluation of the misses =================
        bool all_dead = false;
        if (!kTC) {
            if (!own_alive) break;
            const int nmiss = c.nmiss;
            // memo insert, part 1: way 1 <- way 0, way 0 key <- window (the evaluator fills way 0's rates)
            for (int q = warp; q < nmiss; q += kWarps) {
                const int r = c.miss[q];
                MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                uint4 t = make_uint4(0, 0, 0, 0);
                if (lane < 9) t = reinterpret_cast<const uint4*>(&me[0])[lane];
                __syncwarp();
                if (lane < 9) reinterpret_cast<uint4*>(&me[1])[lane] = t;
                __syncwarp();
                if (lane < 16) reinterpret_cast<uint32_t*>(me[0].key)[lane] = reinterpret_cast<const uint32_t*>(win + r * kWin)[lane];
                if (lane == 0) c.row_way[r] = 0;
            }
            __syncthreads();
            if (!mlp) {
                for (int q = tid; q < nmiss; q += kThreads) {
                    const int r = c.miss[q];
                    const uint8_t* w = win + r * kWin;
                    MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                    const int vox = c.mem_vac[c.row_mem[r]].x;
                    double R = 0.0;
                    int cl = 0;
                    for (int k = 0; k < kHops; ++k) {
                        double E = 0.0, Gk = 0.0;
                        if (w[k] != kVac) {
                            cl += pair_barrier(w, k, p.G, p.P, E);
                            Gk = arrhenius(E, p.P, vox);
                        }
                        R = __dadd_rn(R, Gk);
                        me[0].G[k] = Gk;
                    }
                    rowR[r] = R;
                    rowC[r] = cl;
                    me[0].R = R;
                    me[0].clamps = cl;
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
                        MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                        const int vox = c.mem_vac[c.row_mem[r]].x;
                        double R = 0.0;
                        for (int k = 0; k < kHops; ++k) {
                            const double Gk = (w[k] != kVac) ? arrhenius(Ek[k], p.P, vox) : 0.0;
                            R = __dadd_rn(R, Gk);
                            me[0].G[k] = Gk;
                        }
                        rowR[r] = R;
                        rowC[r] = 0;
                        me[0].R = R;
                        me[0].clamps = 0;
                    }
                    __syncthreads();
                }
            }
            __syncthreads();
        } else {
            // ---- FP32-equivalent evaluator: rounds in lockstep over the cluster
            if (phase_mode) {
                // memo insert, part 1, for every miss of this iteration: way 1 <- way 0, way 0 key <- window
                // (E3 fills way 0's rates); a warp moves kEL1Rows entries at a time
                const int nmiss = c.nmiss;
                for (int q0 = warp; q0 < nmiss; q0 += kEL1Rows * kWarps) {
                    MemoEntry* me[kEL1Rows];
                    uint4 tm[kEL1Rows];
                    uint32_t kw[kEL1Rows];
#pragma unroll
                    for (int q = 0; q < kEL1Rows; ++q) {
                        const int qq = q0 + q * kWarps;
                        tm[q] = make_uint4(0, 0, 0, 0);
                        kw[q] = 0;
                        me[q] = nullptr;
                        if (qq < nmiss) {
                            const int r = c.miss[qq];
                            me[q] = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                            if (lane < 9) tm[q] = reinterpret_cast<const uint4*>(&me[q][0])[lane];
                            if (lane < 16) kw[q] = reinterpret_cast<const uint32_t*>(win + r * kWin)[lane];
                        }
                    }
#pragma unroll
                    for (int q = 0; q < kEL1Rows; ++q)
                        if (me[q] && lane < 9) reinterpret_cast<uint4*>(&me[q][1])[lane] = tm[q];
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < kEL1Rows; ++q)
                        if (me[q] && lane < 16) reinterpret_cast<uint32_t*>(me[q][0].key)[lane] = kw[q];
                }
            }
            if (tid == 0) lap(d_y[0]);
            int k_round = 0;
            for (;;) {
                int own_n = 0;
                if (phase_mode) {
                    own_n = min(kRoundRows, max(0, c.nmiss - kRoundRows * k_round));
                    // layer 1 of this round's own rows (two per warp at a time); memo way 1 <- way 0, key <- window
                    for (int i = warp; i < own_n; i += kEL1Rows * kWarps) {
                        const int nv = min(kEL1Rows, (own_n - i + kWarps - 1) / kWarps);
                        int rr[kEL1Rows], mr[kEL1Rows];
#pragma unroll
                        for (int q = 0; q < kEL1Rows; ++q) {
                            rr[q] = c.miss[kRoundRows * k_round + (q < nv ? i + q * kWarps : i)];
                            mr[q] = kRoundRows * (int)rank + i + q * kWarps;
                        }
                        layer1_rows<kEL1Rows, kEL1Batch>(rr, nv, win, l1n, l1l, p.W.W1f, mr, A_hi, A_lo, g_hi, g_lo, ovf,
                                                         fast, p.W.h1s,
                                    (AKMC_L1_PROBE && tid == 0 && p.diag) ? d_z : nullptr);
                    }
                    if (tid == 0) {
                        hdr[rank].n = own_n;
                        hdr[rank].more = (c.nmiss > kRoundRows * (k_round + 1)) ? 1 : 0;
                        hdr[rank].alive = own_alive;
                    }
                } else {
                    // eval mode: the next 16 rows from the cursor; windows into win[0..16)
                    __syncthreads();
                    if (tid == 0) c.ebase = (int)atomicAdd(p.cursor, (unsigned)kRoundRows);
                    __syncthreads();
                    const int base = c.ebase;
                    own_n = min(kRoundRows, max(0, nrows_eval - base));
                    for (int i = warp; i < own_n; i += kWarps) {
                        const int g = base + i;
                        uint8_t a0, a1;
                        if (p.windows) {
                            a0 = p.windows[(size_t)g * kWin + lane];
                            a1 = p.windows[(size_t)g * kWin + lane + 32];
                        } else {
                            const int slot = p.rows ? p.rows[g] : g;
                            const int4 v = p.vac[slot];
                            const bool live = v.x >= 0;                 // departed slot (multi-rank): any window
                            a0 = live ? site_byte_pk(p.species, p.F, v, off_lo) : (uint8_t)kFe;
                            a1 = live ? site_byte_pk(p.species, p.F, v, off_hi) : (uint8_t)kFe;
                        }
                        win[i * kWin + lane] = a0;
                        win[i * kWin + lane + 32] = a1;
                        if (lane < 8) win8[i * 8 + lane] = a0;
                        l1_list_store(i, a0, a1, l1n, l1l);
                    }
                    __syncwarp();
                    for (int i = warp; i < own_n; i += kEL1Rows * kWarps) {
                        const int nv = min(kEL1Rows, (own_n - i + kWarps - 1) / kWarps);
                        int rr[kEL1Rows], mr[kEL1Rows];
#pragma unroll
                        for (int q = 0; q < kEL1Rows; ++q) {
                            rr[q] = q < nv ? i + q * kWarps : i;
                            mr[q] = kRoundRows * (int)rank + i + q * kWarps;
                        }
                        layer1_rows<kEL1Rows, kEL1Batch>(rr, nv, win, l1n, l1l, p.W.W1f, mr, A_hi, A_lo, g_hi, g_lo, ovf,
                                                         fast, p.W.h1s,
                                    (AKMC_L1_PROBE && tid == 0 && p.diag) ? d_z : nullptr);
                    }
                    if (tid == 0) { hdr[rank].n = own_n; hdr[rank].more = 0; hdr[rank].alive = own_n > 0 ? 1 : 0; }
                }
                wd(4, k_round, own_n);
                if (tid == 0) lap(d_y[1]);
                // ---- exchange: header (DSMEM) + this CTA's h1 rows (8-row groups 4r..4r+3), multicast from the
                //      L2 staging copy into every peer's A (one L2 read, no SM-to-SM bandwidth limit)
                fence_async_smem();
#if !AKMC_XCHG_DSMEM
                fence_async_global();
#endif
                __syncthreads();
                if (tid == 0) lap(d_y[2]);
                if (warp == 0 && lane < kClusterN) {        // lane d signals CTA d
                    const uint32_t d = (uint32_t)lane;
                    const uint32_t rg = (uint32_t)((own_n + 7) >> 3);
#if AKMC_XCHG_DSMEM
                    // h1 rows straight from this CTA's A into each peer's A (SM-to-SM, no L2 round trip)
                    if (d == rank) {
                        mbar_arrive(bar_req);
                    } else {
                        const uint32_t cb = map_to(bar_req, d);
                        const uint32_t aoff = (uint32_t)(kRoundRows / 8) * rank * kRowGroupA;
                        mbar_remote_expect_tx(cb, 16u + 2u * rg * kRowGroupA);
                        bulk_s2peer(map_to(smem_u32(&hdr[rank]), d), smem_u32(&hdr[rank]), 16u, cb);
                        if (rg) {
                            bulk_s2peer(map_to(smem_u32(A_hi + aoff), d), smem_u32(A_hi + aoff), rg * kRowGroupA, cb);
                            bulk_s2peer(map_to(smem_u32(A_lo + aoff), d), smem_u32(A_lo + aoff), rg * kRowGroupA, cb);
                        }
                    }
#else
                    if (d == rank) {
                        mbar_arrive(bar_req);
                        if (rg) {
                            const uint32_t aoff = (uint32_t)(kRoundRows / 8) * rank * kRowGroupA;
                            const uint16_t mask = (uint16_t)(((1u << kClusterN) - 1u) & ~(1u << rank));
                            bulk_g2s_multicast(smem_u32(A_hi + aoff), g_hi, rg * kRowGroupA, bar_req, mask);
                            if (!fast) bulk_g2s_multicast(smem_u32(A_lo + aoff), g_lo, rg * kRowGroupA, bar_req, mask);
                        }
                    } else {
                        const uint32_t cb = map_to(bar_req, d);
                        mbar_remote_expect_tx(cb, 16u + (fast ? 1u : 2u) * rg * kRowGroupA);
                        bulk_s2peer(map_to(smem_u32(&hdr[rank]), d), smem_u32(&hdr[rank]), 16u, cb);
                    }
#endif
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                mbar_wait_cluster(bar_req, ph_req);
                ph_req ^= 1u;
#if AKMC_XCHG_DSMEM
                // the outgoing copies read this CTA's row block, which E2 overwrites with h2
                if (warp == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
                wd(5, k_round, own_n);
                if (tid == 0) { const long long before = d_x[4]; lap(d_x[4]); if (k_round > 0) d_xk += d_x[4] - before; }
                int n_s[kClusterN];
                int any_more = 0, any_alive = 0, total = 0;
#pragma unroll
                for (int s = 0; s < kClusterN; ++s) {
                    n_s[s] = hdr[s].n;
                    any_more |= hdr[s].more;
                    any_alive |= hdr[s].alive;
                    total += hdr[s].n;
                }
                if (k_round == 0 && !any_alive) all_dead = true;
                if (total > 0) {
                    // ---- L2 on tcgen05: D1 (TMEM cols [0, 64)), D2 (cols [64, 128))
                    tc_fence_before();
                    __syncthreads();
                    tc_fence_after();
                    if (tid == 0) {
                        const uint32_t idesc = idesc_f16(kTileRows, kSliceN);
                        const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo), wb = smem_u32(sm + kOffW2);
                        for (int ks = 0; ks < kHid / 16; ++ks) {
                            const uint64_t dah = umma_desc(ah + (uint32_t)ks * 256u, 128, kRowGroupA);
                            const uint64_t dal = umma_desc(al + (uint32_t)ks * 256u, 128, kRowGroupA);
                            const uint64_t dbh = umma_desc(wb + (uint32_t)ks * 2u * kW2Split, (kSliceN / 8) * 128, 128);
                            const uint64_t dbl = umma_desc(wb + (uint32_t)ks * 2u * kW2Split + kW2Split, (kSliceN / 8) * 128, 128);
                            umma_f16(tmem + 0, dah, dbh, idesc, ks > 0 ? 1u : 0u);
                            if (!fast) {
                                umma_f16(tmem + kSliceN, dah, dbl, idesc, ks > 0 ? 1u : 0u);
                                umma_f16(tmem + kSliceN, dal, dbh, idesc, 1u);
                            }
                        }
                        umma_commit(bar_mma);
                    }
                    mbar_wait(bar_mma, ph_mma);
                    ph_mma ^= 1u;
                    tc_fence_after();
                    // ---- E2 + layer 3 (FP64, CUDA cores): warp = (TMEM lane quadrant q4 = source block, 32-column
                    //      half hc); a thread holds one row and 2 chunks of 16 h2 columns: P_q, their pair sum
                    {
                        const int q4 = warp & 3, hc = warp >> 2;
                        const int m = 32 * q4 + lane;
                        const bool rows_here = quad_has_rows(n_s, q4);
                        double pr[8];
                        if (rows_here) {
                            const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
                            const double* w3s = reinterpret_cast<const double*>(sm + kOffW3);
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                const int c0 = 32 * hc + 16 * hh;
                                uint32_t d1[16], d2[16];
                                tmem_ld16(tl + (uint32_t)c0, d1);
                                if (!fast) tmem_ld16(tl + (uint32_t)(kSliceN + c0), d2);
                                else
#pragma unroll
                                    for (int t = 0; t < 16; ++t) d2[t] = 0u;
                                tmem_wait_ld();
                                float z[16];
                                e2_chunk(d1, d2, b2s + c0, p.W.s2u, z);
                                double P[8];
                                l3_chunk(z, w3s + c0 * 8, P);
#pragma unroll
                                for (int k = 0; k < 8; ++k) pr[k] = hh ? __dadd_rn(pr[k], P[k]) : P[k];
                            }
                            if (hc == 1) {
                                double2* dst = reinterpret_cast<double2*>(pair_tmp + m * 8);
                                dst[0] = make_double2(pr[0], pr[1]); dst[1] = make_double2(pr[2], pr[3]);
                                dst[2] = make_double2(pr[4], pr[5]); dst[3] = make_double2(pr[6], pr[7]);
                            }
                        }
                        tc_fence_before();
                        __syncthreads();
                        if (rows_here && hc == 0) {
                            const double2* o = reinterpret_cast<const double2*>(pair_tmp + m * 8);
                            double2* dst = reinterpret_cast<double2*>(part_out + m * 8);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const double2 b = o[j];
                                dst[j] = make_double2(__dadd_rn(pr[2 * j], b.x), __dadd_rn(pr[2 * j + 1], b.y));
                            }
                        }
                    }
                    if (tid == 0) lap(d_x[5]);
                    // ---- partials of row block s -> CTA s (every CTA arrives on every CTA's barrier)
                    fence_async_smem();
                    tc_fence_before();
                    __syncthreads();
                    if (warp == 0 && lane < kClusterN) {    // lane s sends row block s to CTA s
                        const uint32_t s = (uint32_t)lane;
                        const uint32_t bytes = (uint32_t)n_s[s] * 64u;
                        const uint32_t cb = map_to(bar_part, s);
                        mbar_remote_expect_tx(cb, bytes);
                        if (bytes)
                            bulk_s2peer(map_to(smem_u32(part_in + rank * kRoundRows * 8), s),
                                        smem_u32(part_out + s * kRoundRows * 8), bytes, cb);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    wd(6, k_round, own_n);
                    mbar_wait_cluster(bar_part, ph_part);
                    ph_part ^= 1u;
                    wd(7, k_round, own_n);
                    if (tid == 0) lap(d_x[6]);
                    // ---- E3 for this CTA's own rows: thread (row i, hop k)
                    if (tid < kRoundRows * 8) {
                        const int i = tid >> 3, k = tid & 7;
                        const bool valid = i < own_n;
                        const int r = phase_mode ? (valid ? (int)c.miss[kRoundRows * k_round + i] : 0) : i;
                        double Gk = 0.0, Ek = 0.0;
                        if (valid) {
                            double acc = 0.0;
#pragma unroll
                            for (int s = 0; s < kClusterN; ++s) acc = __dadd_rn(acc, part_in[(s * kRoundRows + i) * 8 + k]);
                            const double out = __dadd_rn(b3s[k], acc);
                            Ek = out > 0.0 ? out : 0.0;
                            int vox = -1;
                            if (phase_mode) vox = c.mem_vac[c.row_mem[r]].x;
                            else if (!p.windows) vox = max(p.vac[p.rows ? p.rows[c.ebase + i] : c.ebase + i].x, 0);
                            Gk = (win8[r * 8 + k] != (uint8_t)kVac) ? arrhenius_tc(Ek, p.P, vox) : 0.0;
                        }
                        double R = 0.0;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) R = __dadd_rn(R, __shfl_sync(0xffffffffu, Gk, (lane & ~7) + kk));
                        if (valid) {
                            if (phase_mode) {
                                MemoEntry* me = p.memo + 2 * (size_t)c.mem_slot[c.row_mem[r]];
                                me[0].G[k] = Gk;
                                if (k == 0) { rowR[r] = R; c.row_way[r] = 0; me[0].R = R; me[0].clamps = 0; }
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
                if (warp == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (tid == 0) {
                    lap(d_x[7]);
                    ++d_rounds;
                    d_erounds += total > 0 ? 1 : 0;
                }
                __syncthreads();
                ++k_round;
                if (!any_more) break;
            }
            if (all_dead) break;
            if (!phase_mode) continue;
        }

        // ================= BKL step per running domain (thread per head slot) =================
        __syncthreads();
        wd(9, 0, 0);
        if (tid == 0) lap(d_cr);
        if (tid < kSlots && c.seg_used[tid] == 1 && c.seg_run[tid]) {
            const int i = tid;
            const int cnt = c.seg_cnt[i], moff = kSlotCap * i;
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
                    if (!kTC) cl += (unsigned long long)rowC[r];
                    idx[m] = a;
                    ++m;
                }
            bool stop = false;
            if (m == 0) {
                stop = true;
                if (p.serial) {                               // a voxel without vacancies: terminal
                    p.term[c.seg_dom[i]] = 1;
                    atomicAdd(&p.ctr->terminal, 1ull);
                }
            } else {
                my_evals += 8ull * (unsigned long long)m;
                my_clamps += cl;
                int P = 1, nlev = 0;
                const double Rd = tree_build(buf, m, P, nlev);
                if (!(Rd > 0.0)) {
                    stop = true;
                    if (p.serial) {                           // no feasible event in this voxel
                        p.term[c.seg_dom[i]] = 1;
                        p.nev[c.seg_dom[i]] += c.seg_it[i];
                        atomicAdd(&p.ctr->terminal, 1ull);
                    }
                } else {
                    // Memo-hit chain (R7 + R6): a domain with ONE active member is the only writer of the sites its
                    // windows read in this phase (A20; the other members do not move), so after its hop the next
                    // iteration would gather exactly the window the hop left.  If that window is already a key of
                    // the vacancy's memo (a back-hop restores an earlier configuration exactly), the next
                    // iteration would be a pure memo hit and its BKL step can run here at once, with the same
                    // Philox counter (the domain's own event index) -- bit-identical to waiting for the
                    // iteration, without its gather + evaluation round.  The window comparison is the full
                    // 64-byte key, so nothing is assumed about which configuration recurs.
                    double u_sel, u_t, dt;
                    bool go;
                    double Rc = Rd;
                    const MemoEntry* src = nullptr;      // chained step: the memo way that holds the rates
                    int a = 0;
                    const bool may_chain = m == 1 && AKMC_CHAIN_MAX > 0 && c.nrun <= AKMC_CHAIN_NRUN;
                    for (int chain = 0;; ++chain) {
                    if (p.serial) {
                        // serial BKL (a10): counter (event index of the voxel, voxel), clock += dt after the hop
                        const unsigned long long n = (unsigned long long)p.nev[c.seg_dom[i]] + c.seg_it[i];
                        philox_uniforms(p.S.seed, make_uint4((uint32_t)n, (uint32_t)(n >> 32), c.seg_dom[i], 0u), u_sel, u_t);
                        dt = __ddiv_rn(-det_log(u_t), Rc);
                        go = !(p.horizon && __dadd_rn(AKMC_SERIAL_CLOCK ? c.seg_t[i] : p.clock[c.seg_dom[i]], dt) > p.t_end);
                    } else {
                        const unsigned long long ph = (unsigned long long)p.ph[c.seg_q[i]].phase;
                        philox_uniforms(p.S.seed, make_uint4(c.seg_it[i], (uint32_t)c.seg_dom[i], (uint32_t)ph, (uint32_t)(ph >> 32)),
                                        u_sel, u_t);
                        dt = __ddiv_rn(-det_log(u_t), Rc);
                        go = !(__dadd_rn(c.seg_t[i], dt) > p.S.window);   // else the overshooting draw is discarded
                    }
                    if (!go) {
                        stop = true;
                        if (p.serial) p.nev[c.seg_dom[i]] += c.seg_it[i];   // horizon reached in this launch
                        break;
                    } else {
                        double rr = __dmul_rn(u_sel, Rc);
                        if (chain == 0) a = idx[tree_descend(buf, m, P, nlev, rr)];   // m == 1 in a chain: rr as is
                        const int slot = c.mem_slot[moff + a];
                        const int r = c.mem_row[moff + a];
                        const MemoEntry& mrow = chain ? *src : p.memo[2 * (size_t)slot + c.row_way[r]];   // the rates
                        const int k = pick_hop(mrow.G, rr);
                        // hop: the target's species is window slot k (1NN slots are 0..7)
                        const int4 ov = c.mem_vac[moff + a];
                        int4 nv = ov;
                        nv.y = p.F.wrap[0] ? wrap2(ov.y + p.G.off[k][0], 2 * p.F.L[0]) : ov.y + p.G.off[k][0];
                        nv.z = p.F.wrap[1] ? wrap2(ov.z + p.G.off[k][1], 2 * p.F.L[1]) : ov.z + p.G.off[k][1];
                        nv.w = p.F.wrap[2] ? wrap2(ov.w + p.G.off[k][2], 2 * p.F.L[2]) : ov.w + p.G.off[k][2];
                        const uint8_t tn = chain ? mrow.key[k] : win8[r * 8 + k];
                        write_site(p.species, p.F, ov.x, ov.y, ov.z, ov.w, tn);
                        write_site(p.species, p.F, nv.x, nv.y, nv.z, nv.w, (uint8_t)kVac);
#if AKMC_PREFETCH
                        prefetch_vacancy(p.species, p.F, nv, p.memo + 2 * (size_t)slot);
#endif
                        p.vac[slot] = nv;
                        c.mem_vac[moff + a] = nv;
                        long long d2 = 0;
                        int sec2 = 0;
                        if (!p.serial) dom_sector(nv, p.S, d2, sec2);
                        if (!p.serial && (d2 != (long long)c.seg_dom[i] || sec2 != p.ph[c.seg_q[i]].sector)) c.mem_act[moff + a] = 0;
                        if (kDF) {
                            // a vacancy entering another tile is announced to it (read at that tile's next activation)
                            const int Tn = df_tile_of(p, d2);
                            if (Tn != df_tile_of(p, (long long)c.seg_dom[i])) {
                                const int k2 = atomicAdd(p.arr_cnt + Tn, 1);
                                if (k2 < kArrCap) p.arr_slot[(size_t)Tn * kArrCap + k2] = slot;
                                else atomicAdd(p.df_err, 1);
                            }
                        }
                        if (p.S.log) {
                            if (near_face(p.F, ov.y, ov.z, ov.w))
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, ov.y, ov.z, ov.w, tn);
                            if (near_face(p.F, nv.y, nv.z, nv.w))
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, nv.y, nv.z, nv.w, kVac);
                            bool out = false;
                            const int np[3] = {nv.y, nv.z, nv.w};
                            for (int ax = 0; ax < 3; ++ax)
                                if (!p.F.wrap[ax] && (np[ax] < 0 || np[ax] >= 2 * p.F.L[ax])) out = true;
                            if (out) {
                                log_entry(p.S.log, p.S.nlog, p.S.logcap, nv.y, nv.z, nv.w, kMigrateBase + p.S.gid[slot]);
                                depart_slot(p.vac, p.S, slot);
                            }
                        }
                        c.seg_t[i] = __dadd_rn(c.seg_t[i], dt);
                        c.seg_it[i] += 1u;
                        my_events += 1ull;
                        if (p.serial) {
                            const unsigned v = c.seg_dom[i];
                            p.clock[v] = AKMC_SERIAL_CLOCK ? c.seg_t[i] : __dadd_rn(p.clock[v], dt);
                            if ((int)c.seg_it[i] >= p.n_events) {   // this launch's events done
                                p.nev[v] += c.seg_it[i];
                                stop = true;
                            }
                        }
                        // ---- chain test: is the window the hop left a key of the vacancy's memo?
                        if (stop || !may_chain || chain >= AKMC_CHAIN_MAX || !c.mem_act[moff + a] || p.vac[slot].x < 0) break;
                        my_check += 1ull;
                        uint32_t ww[kWin / 4];
                        // stage 1: the 8 first-shell bytes against both ways (most failing checks end here)
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            uint32_t wq = 0;
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                wq |= (uint32_t)p.species[neighbour_site(p.F, nv, p.G.off[4 * q + j][0], p.G.off[4 * q + j][1],
                                                                         p.G.off[4 * q + j][2])] << (8 * j);
                            ww[q] = wq;
                        }
                        {
                            const uint2 k0 = *reinterpret_cast<const uint2*>(p.memo[2 * (size_t)slot].key);
                            const uint2 k1 = *reinterpret_cast<const uint2*>(p.memo[2 * (size_t)slot + 1].key);
                            if (!((k0.x == ww[0] && k0.y == ww[1]) || (k1.x == ww[0] && k1.y == ww[1]))) break;
                        }
#pragma unroll
                        for (int q = 2; q < kWin / 4; ++q) {
                            uint32_t wq = 0;
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                wq |= (uint32_t)p.species[neighbour_site(p.F, nv, p.G.off[4 * q + j][0], p.G.off[4 * q + j][1],
                                                                         p.G.off[4 * q + j][2])] << (8 * j);
                            ww[q] = wq;
                        }
                        int hw = -1;
#pragma unroll
                        for (int w = 0; w < 2; ++w) {
                            const uint4* kq = reinterpret_cast<const uint4*>(p.memo[2 * (size_t)slot + w].key);
                            bool eq = true;
#pragma unroll
                            for (int q = 0; q < kWin / 16; ++q) {
                                const uint4 t = kq[q];
                                eq = eq && t.x == ww[4 * q] && t.y == ww[4 * q + 1] && t.z == ww[4 * q + 2] && t.w == ww[4 * q + 3];
                            }
                            if (eq && hw < 0) hw = w;
                        }
                        if (hw < 0) break;
                        src = &p.memo[2 * (size_t)slot + hw];
                        Rc = src->R;
                        if (!(Rc > 0.0)) break;                  // the next iteration handles a dead vacancy
                        // the chained step is one more logical evaluation of this vacancy (R4 accounting)
                        my_evals += 8ull;
                        if (!kTC) my_clamps += (unsigned long long)src->clamps;
                        my_chain += 1ull;
                    }
                    }
                }
            }
            if (stop) {
                c.seg_run[i] = 0;
                if (kDF && atomicSub(&c.df_left[c.seg_tp[i]], 1) == 1)    // the tile's phase is complete
                    st_release_gpu_s64(p.done_phase + c.df_tile[c.seg_tp[i]], p.ph[c.seg_q[i]].phase);
            }
        }
        __syncthreads();
        if (tid == 0) lap(d_cs);
        trace_end();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // (the next phase's activation may launch)
    if (tid == 0 && p.diag && phase_mode) atomicAdd(p.diag + 96 + 512 + min(tr_it, 63), 1ull);
    if (tid == 0 && p.diag && p.overlap) {
        // overlap timing: boundary list publication and engine end, relative to the engine's start (last CTA out)
        __threadfence();
        if (atomicAdd(&p.ctr->nexit, 1ull) == gridDim.x - 1) {
            long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            const long long e0 = *(volatile long long*)&p.ctr->t_e0, tp = *(volatile long long*)&p.ctr->t_pub;
            atomicAdd(p.diag + 88, (unsigned long long)max(0ll, tp - e0));
            atomicAdd(p.diag + 89, (unsigned long long)max(0ll, now - e0));
            atomicAdd(p.diag + 90, 1ull);
            atomicAdd(p.diag + 91, tp < e0 ? 1ull : 0ull);
        }
    }
    if (tid == 0 && p.diag) {
        d_cc = d_x[0] + d_x[1] + d_x[2];
        d_x[3] = d_y[0] + d_y[1] + d_y[2];
        d_cr += d_x[3] + d_x[4] + d_x[5] + d_x[6] + d_x[7];
        atomicAdd(p.diag + 0, d_it);
        atomicMax(p.diag + 1, d_it);
        atomicAdd(p.diag + 2, d_rounds);
        atomicAdd(p.diag + 3, d_erounds);
        atomicAdd(p.diag + 4, (unsigned long long)d_cc);
        atomicAdd(p.diag + 5, (unsigned long long)d_cr);
        atomicAdd(p.diag + 6, (unsigned long long)d_cs);
        atomicAdd(p.diag + 7, 1ull);
        atomicAdd(p.diag + 8, d_refill);
        atomicAdd(p.diag + 9, (unsigned long long)(clock64() - t_start));
        atomicAdd(p.diag + 10, 1ull * (phase_mode ? 1 : 0));
        for (int q = 0; q < 8; ++q) atomicAdd(p.diag + 11 + q, (unsigned long long)d_x[q]);
        for (int q = 0; q < 3; ++q) atomicAdd(p.diag + 20 + q, (unsigned long long)d_y[q]);
        for (int q = 0; q < 4; ++q) atomicAdd(p.diag + 24 + q, (unsigned long long)d_z[q]);
        atomicAdd(p.diag + 19, (unsigned long long)d_xk);
        for (int q = 0; q < 4; ++q) atomicAdd(p.diag + 56 + q, (unsigned long long)d_df[q]);
    }

    // ---- teardown
    if (ovf && p.overflow) atomicAdd(p.overflow, ovf);
    if (phase_mode && tid < 32 * kMaskWords) {   // whole warps (slot threads are tid < kSlots)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            my_events += __shfl_xor_sync(0xffffffffu, my_events, o);
            my_evals += __shfl_xor_sync(0xffffffffu, my_evals, o);
            my_clamps += __shfl_xor_sync(0xffffffffu, my_clamps, o);
            my_chain += __shfl_xor_sync(0xffffffffu, my_chain, o);
            my_check += __shfl_xor_sync(0xffffffffu, my_check, o);
        }
        if (lane == 0 && p.diag && my_chain) atomicAdd(p.diag + 29, my_chain);
        if (lane == 0 && p.diag && my_check) atomicAdd(p.diag + 30, my_check);
        if (lane == 0) { atomicAdd(&c.events, my_events); atomicAdd(&c.evals, my_evals); atomicAdd(&c.clamps, my_clamps); }
    }
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
            tmem_dealloc(tmem, 256);
        }
    }
}

// ---- dataflow sweep preparation: every tile's vacancies at the start of the sweep (base lists), no arrivals yet,
//      done_phase = the phase before the sweep's first
__global__ void df_count_kernel(const int4* __restrict__ vac, int nv, EngineParams p, int* cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < p.ntiles) { p.arr_cnt[i] = 0; p.done_phase[i] = p.ph[0].phase - 1; }
    if (i >= nv) return;
    const int4 v = vac[i];
    if (v.x < 0) return;
    long long d; int sec;
    dom_sector(v, p.S, d, sec);
    atomicAdd(cnt + df_tile_of(p, d), 1);
}
__global__ void __launch_bounds__(1024) df_scan_kernel(const int* cnt, int n, int* off, int* cursor)
{
    // single block: exclusive scan of n counts (n <= a few 1e4)
    __shared__ int part[1024];
    const int per = (n + 1023) / 1024;
    const int b = threadIdx.x * per;
    int sum = 0;
    for (int k = 0; k < per && b + k < n; ++k) sum += cnt[b + k];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int t = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += t;
        __syncthreads();
    }
    int run = part[threadIdx.x] - sum;
    for (int k = 0; k < per && b + k < n; ++k) { off[b + k] = run; cursor[b + k] = run; run += cnt[b + k]; }
    if (threadIdx.x == 1023) off[n] = part[1023];
}
__global__ void df_scatter_kernel(const int4* __restrict__ vac, int nv, EngineParams p, int* cursor, int* mem)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const int4 v = vac[i];
    if (v.x < 0) return;
    long long d; int sec;
    dom_sector(v, p.S, d, sec);
    mem[atomicAdd(cursor + df_tile_of(p, d), 1)] = i;
}

} // namespace

cudaError_t launch_df_prep(const EngineParams& p, const int4* vac, int nv, int* cnt, int* off, int* cursor, int* mem,
                           cudaStream_t s)
{
    cudaMemsetAsync(cnt, 0, (size_t)p.ntiles * sizeof(int), s);
    const int n = std::max(nv, p.ntiles);
    df_count_kernel<<<(n + 255) / 256, 256, 0, s>>>(vac, nv, p, cnt);
    df_scan_kernel<<<1, 1024, 0, s>>>(cnt, p.ntiles, off, cursor);
    df_scatter_kernel<<<(nv + 255) / 256, 256, 0, s>>>(vac, nv, p, cursor, mem);
    return cudaGetLastError();
}

size_t engine_smem_bytes() { return kSmemTotal; }

cudaError_t engine_setup()
{
    const int b = (int)kSmemTotal;
    cudaError_t e = cudaFuncSetAttribute(engine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(engine_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(engine_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(engine_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(engine_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(engine_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    return e;
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
        if (p.df) engine_kernel<false, false, true><<<num_sms, kThreads, kSmemTotal, s>>>(p);
        else engine_kernel<false><<<num_sms, kThreads, kSmemTotal, s>>>(p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterN;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue overlaps the previous kernel
    attr[1].val.programmaticStreamSerializationAllowed = AKMC_PDL;
    cfg.gridDim = dim3(kClusterN * nclusters, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemTotal;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (p.df) return p.fast ? cudaLaunchKernelEx(&cfg, engine_kernel<true, true, true>, p)
                            : cudaLaunchKernelEx(&cfg, engine_kernel<true, false, true>, p);
    return p.fast ? cudaLaunchKernelEx(&cfg, engine_kernel<true, true>, p) : cudaLaunchKernelEx(&cfg, engine_kernel<true>, p);
}

} // namespace akmc
