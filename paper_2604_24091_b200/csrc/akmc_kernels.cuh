// akmc_kernels.cuh -- FP64 evaluation, BKL selection/apply, sublattice bookkeeping and lattice-scan
// kernels of the B200 AKMC path.
//
// Steps of SURVEY sec. 8(a): a0 vacancy registry (device scan), a1 activation/compaction, a2+a3
// gather/encode (FP64 paths), a4' pair KRA / a4 FP64 MLP (verify precision), a5 rates, a6 per-domain
// pairwise tree + Philox draw, a7 apply, a8 inner loop condition, a10 serial/voxel-batch variant.
// Operation order = DESIGN.md sec. 5.  Kernels that run inside the per-sweep CUDA graph read their
// per-phase parameters from device memory (PhaseInfo) and their sizes from device counters, and use
// grid-stride loops, so one graph serves every sweep.
#pragma once
#include <climits>
#include "akmc_device.cuh"
#include "akmc_dist.cuh"

namespace akmc {

struct DevCounters {                 // device-side counters (unsigned long long for atomics)
    unsigned long long events, hop_evals, clamps, terminal, nrun, nseg, total, nrows;
    unsigned long long chunk;        // phase engine: next segment to hand out (reset per phase)
    unsigned long long mrows;        // barrier-network rows actually evaluated (memo misses)
    unsigned long long nhot, ncold;  // phase engine: segments at the front (hot) / back (cold) of the list
    // multi-rank overlap (akmc_api.cu step_sublattice): the boundary domains' segments, built after the previous
    // phase's halo deltas arrived, their cursor, and the phase number they were published for (release / acquire)
    unsigned long long nseg2, chunk2;
    long long bready;
    unsigned long long nbdom;       // multi-rank overlap: boundary domains holding active vacancies (listed)
    long long t_e0, t_pub;          // (AKMC_PHASE_TIMING) globaltimer at the engine's start / at the publication
    unsigned long long nexit;       //   and the engine CTAs that have exited
};

// memo layout as seen from the segment builder (MemoEntry lives in akmc_engine.cuh; asserted there)
constexpr int kMemoBytes = 144, kMemoROff = 128;

// ------------------------------------------------------------------ window gather
__device__ __forceinline__ void gather_window(const uint8_t* __restrict__ species, const Frame& F, const GeomTables& G,
                                              const int4& v, uint8_t (&w)[kWin])
{
#pragma unroll
    for (int j = 0; j < kWin; ++j) w[j] = __ldg(species + neighbour_site(F, v, G.off[j][0], G.off[j][1], G.off[j][2]));
}

__device__ __forceinline__ int row_count(const int* nrows_dev, int nrows_host)
{
    return nrows_dev ? *nrows_dev : nrows_host;
}

// ------------------------------------------------------------------ pair KRA, FP64 (thread per row)
static __global__ void eval_pair_kernel(const uint8_t* __restrict__ species, const int4* __restrict__ vac,
                                 const uint8_t* __restrict__ windows, Frame F, GeomTables G, PhysParams P,
                                 const int* __restrict__ rows, const int* __restrict__ nrows_dev, int nrows_host,
                                 double* __restrict__ rates, double* __restrict__ Rsum, double* __restrict__ Eout,
                                 DevCounters* ctr)
{
    const int nrows = row_count(nrows_dev, nrows_host);
    int clamps = 0;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nrows; g += gridDim.x * blockDim.x) {
        uint8_t w[kWin];
        int slot;
        if (windows) {
            slot = g;
#pragma unroll
            for (int j = 0; j < kWin; ++j) w[j] = windows[(size_t)g * kWin + j];
        } else {
            slot = rows ? rows[g] : g;
            const int4 v = vac[slot];
            if (v.x < 0) {                               // departed slot (multi-rank): nothing to evaluate
#pragma unroll
                for (int j = 0; j < kWin; ++j) w[j] = kFe;
            } else {
                gather_window(species, F, G, v, w);
            }
        }
        const int vox = windows ? -1 : max(vac[slot].x, 0);
        double R = 0.0;
#pragma unroll
        for (int k = 0; k < kHops; ++k) {
            double E = 0.0, Gk = 0.0;
            if (w[k] != kVac) {
                clamps += pair_barrier(w, k, G, P, E);
                Gk = arrhenius(E, P, vox);
            }
            R = __dadd_rn(R, Gk);
            if (rates) rates[(size_t)slot * 8 + k] = Gk;
            if (Eout) Eout[(size_t)slot * 8 + k] = E;
        }
        if (Rsum) Rsum[slot] = R;
    }
    if (clamps && ctr) atomicAdd(&ctr->clamps, (unsigned long long)clamps);
}

// ------------------------------------------------------------------ MLP, FP64 (block of 256 per row)
// layer 1 as the embedding bag over the 64 one-hot rows in slot order (== dense fma loop, A8)
static __global__ void __launch_bounds__(256) eval_mlp_fp64_kernel(
    const uint8_t* __restrict__ species, const int4* __restrict__ vac, const uint8_t* __restrict__ windows, Frame F,
    GeomTables G, PhysParams P, const double* __restrict__ mlp, const int* __restrict__ rows,
    const int* __restrict__ nrows_dev, int nrows_host, double* __restrict__ rates, double* __restrict__ Rsum,
    double* __restrict__ Eout)
{
    const int nrows = row_count(nrows_dev, nrows_host);
    __shared__ uint8_t w[kWin];
    __shared__ double h1[kHid];
    __shared__ double h2[kHid];
    __shared__ double Ek[8];
    __shared__ int slot_s;
    const double* W1 = mlp;
    const double* b1 = W1 + 448 * kHid;
    const double* W2 = b1 + kHid;
    const double* b2 = W2 + kHid * kHid;
    const double* W3 = b2 + kHid;
    const double* b3 = W3 + kHid * 8;
    const int j = threadIdx.x;
    for (int g = blockIdx.x; g < nrows; g += gridDim.x) {
        if (j == 0) slot_s = windows ? g : (rows ? rows[g] : g);
        __syncthreads();
        const int slot = slot_s;
        if (j < kWin) {
            if (windows) {
                w[j] = windows[(size_t)g * kWin + j];
            } else {
                const int4 v = vac[slot];
                w[j] = v.x < 0 ? (uint8_t)kFe : __ldg(species + neighbour_site(F, v, G.off[j][0], G.off[j][1], G.off[j][2]));
            }
        }
        __syncthreads();
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
            const int vox = windows ? -1 : max(vac[slot].x, 0);
            double R = 0.0;
            for (int k = 0; k < kHops; ++k) {
                const double Gk = (w[k] != kVac) ? arrhenius(Ek[k], P, vox) : 0.0;
                R = __dadd_rn(R, Gk);
                if (rates) rates[(size_t)slot * 8 + k] = Gk;
                if (Eout) Eout[(size_t)slot * 8 + k] = Ek[k];
            }
            if (Rsum) Rsum[slot] = R;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ canonical pairwise tree (A17)
// leaves buf[0..n) (already written); pads to P = 2^ceil(log2 n) with 0; node = left + right.
__device__ __forceinline__ double tree_build(double* buf, int n, int& P, int& nlev)
{
    P = 1; nlev = 0;
    while (P < n) { P <<= 1; ++nlev; }
    for (int i = n; i < P; ++i) buf[i] = 0.0;
    int off = 0, width = P;
    while (width > 1) {
        for (int i = 0; i < width / 2; ++i) buf[off + width + i] = __dadd_rn(buf[off + 2 * i], buf[off + 2 * i + 1]);
        off += width;
        width >>= 1;
    }
    return buf[off];
}

// descend: go left if r < L else r -= L; guard: a zero leaf -> last positive leaf
__device__ __forceinline__ int tree_descend(const double* buf, int n, int P, int nlev, double& r)
{
    int idx = 0;
    for (int l = nlev; l >= 1; --l) {
        int off = 0;                                   // offset of level l-1: sum_{j < l-1} P >> j
        for (int jj = 0; jj < l - 1; ++jj) off += P >> jj;
        const double left = buf[off + 2 * idx];
        if (r < left) {
            idx = 2 * idx;
        } else {
            r = __dsub_rn(r, left);
            idx = 2 * idx + 1;
        }
    }
    if (idx >= n || !(buf[idx] > 0.0)) {
        int last = -1;
        for (int i = 0; i < n; ++i)
            if (buf[i] > 0.0) last = i;
        idx = last;
    }
    return idx;
}

// first k with r < cumsum_k (sequential), guard: last k with Gamma > 0
__device__ __forceinline__ int pick_hop(const double* G8, double r)
{
    // the 8 rates are read up front (one burst of independent loads; with the early exit inside the scan each
    // load would wait for the previous comparison), then scanned in hop order exactly as before
    double g[kHops];
#pragma unroll
    for (int k = 0; k < kHops; ++k) g[k] = G8[k];
    double cs = 0.0;
#pragma unroll
    for (int k = 0; k < kHops; ++k) {
        cs = __dadd_rn(cs, g[k]);
        if (r < cs) return k;
    }
    int last = -1;
#pragma unroll
    for (int k = 0; k < kHops; ++k)
        if (g[k] > 0.0) last = k;
    return last;
}

// swap vacancy <-> atom at hop k; returns the new position
__device__ __forceinline__ int4 apply_hop(uint8_t* species, int4* vac, int slot, int k, const Frame& F, const GeomTables& G)
{
    const int4 v = vac[slot];
    int4 n = v;
    n.y = F.wrap[0] ? wrap2(v.y + G.off[k][0], 2 * F.L[0]) : v.y + G.off[k][0];   // non-wrap: may enter the halo
    n.z = F.wrap[1] ? wrap2(v.z + G.off[k][1], 2 * F.L[1]) : v.z + G.off[k][1];
    n.w = F.wrap[2] ? wrap2(v.w + G.off[k][2], 2 * F.L[2]) : v.w + G.off[k][2];
    const uint8_t tv = species[site_of(F, v.x, v.y, v.z, v.w)];
    const uint8_t tn = species[site_of(F, n.x, n.y, n.z, n.w)];
    write_site(species, F, v.x, v.y, v.z, v.w, tn);     // owned sites and their ghost images
    write_site(species, F, n.x, n.y, n.z, n.w, tv);
    vac[slot] = n;
    return n;
}

// ------------------------------------------------------------------ serial BKL (a10): thread per voxel
static __global__ void select_serial_kernel(uint8_t* species, int4* vac, Frame F, GeomTables G, int nvox,
                                     const int* __restrict__ vstart, const double* __restrict__ rates,
                                     const double* __restrict__ Rsum, double* scratch, double* clock,
                                     long long* nev, int* term, uint64_t seed, DevCounters* ctr)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvox || term[v]) return;
    const int a0 = vstart[v];
    const int m = vstart[v + 1] - a0;
    atomicAdd(&ctr->hop_evals, 8ull * (unsigned long long)m);
    double* buf = scratch + 4 * (size_t)a0;     // [4*a0, 4*a0 + 4m) holds the 2P-1 tree nodes
    for (int a = 0; a < m; ++a) buf[a] = Rsum[a0 + a];
    int P = 1, nlev = 0;
    const double tot = (m > 0) ? tree_build(buf, m, P, nlev) : 0.0;
    if (!(tot > 0.0)) {
        term[v] = 1;
        atomicAdd(&ctr->terminal, 1ull);
        return;
    }
    const unsigned long long n = (unsigned long long)nev[v];
    double u_sel, u_t;
    philox_uniforms(seed, make_uint4((uint32_t)n, (uint32_t)(n >> 32), (uint32_t)v, 0u), u_sel, u_t);
    double r = __dmul_rn(u_sel, tot);
    const int a = tree_descend(buf, m, P, nlev, r);
    const int k = pick_hop(rates + (size_t)(a0 + a) * 8, r);
    apply_hop(species, vac, a0 + a, k, F, G);
    const double dt = __ddiv_rn(-det_log(u_t), tot);
    clock[v] = __dadd_rn(clock[v], dt);
    nev[v] = (long long)(n + 1);
    atomicAdd(&ctr->events, 1ull);
}

// ------------------------------------------------------------------ sublattice (a1, a6-a8)
struct SubParams {
    int D[3];              // domain edge (cells)
    int ND[3];             // domains per axis per voxel (global: the whole decomposed lattice)
    long long ndom_vox;    // domains per voxel (global)
    double window;         // Delta_win
    uint64_t seed;
    int O[3];              // this rank's block origin (global cells); 0 for a single rank
    int Gc[3];             // global cells per axis (= cells for a single rank)
    const int* gid;        // global slot id per local slot (identity for a single rank)
    // multi-rank: log of writes near non-wrap faces and vacancy departures (akmc_dist.cuh)
    int4* log;
    unsigned long long* nlog;
    int logcap;
    // multi-rank: local slots freed by departures (reused by arrivals, akmc_dist.cuh); fcnt[0] = free count
    int* freelist;
    int* fcnt;
    // multi-rank: local block cells and decomposed axes (a domain within 3 cells of a decomposed face is a
    // "boundary" domain: it reads the halo or receives arrivals; the others are "interior")
    int Lb[3];
    int dec[3];
};

// a vacancy left this rank's block: its local slot is marked departed and pushed on the free list
__device__ __forceinline__ void depart_slot(int4* vac, const SubParams& S, int slot)
{
    vac[slot].x = -1;
    if (S.freelist) S.freelist[atomicAdd(&S.fcnt[0], 1)] = slot;
}

__device__ __forceinline__ int imodk(int a, int m) { const int r = a % m; return r < 0 ? r + m : r; }

struct PhaseInfo {         // per phase, written to device memory before each sweep's graph launch
    int sector;            // active octant c = perm_sweep[q]
    int pad;
    long long phase;       // global phase p = 8*sweep + q
};

struct Segment {
    long long dom;
    int off, cnt;
    double t;
    unsigned int it;
    int running;
};

__device__ __forceinline__ void dom_sector(const int4& v, const SubParams& S, long long& dom, int& sec)
{
    // global cell (the block origin shifts local cells; halo positions wrap around the global torus)
    const int cx = imodk((v.y >> 1) + S.O[0], S.Gc[0]);
    const int cy = imodk((v.z >> 1) + S.O[1], S.Gc[1]);
    const int cz = imodk((v.w >> 1) + S.O[2], S.Gc[2]);
    const int dx = cx / S.D[0], dy = cy / S.D[1], dz = cz / S.D[2];
    const int ox = (cx - dx * S.D[0]) >= (S.D[0] >> 1);
    const int oy = (cy - dy * S.D[1]) >= (S.D[1] >> 1);
    const int oz = (cz - dz * S.D[2]) >= (S.D[2] >> 1);
    dom = (long long)v.x * S.ndom_vox + dx + (long long)S.ND[0] * (dy + (long long)S.ND[1] * dz);
    sec = ox | (oy << 1) | (oz << 2);
}

// part of the domain a vacancy is in: 1 = interior (its phase reads and writes stay >= 3 - 2.5 cells inside the
// block along every decomposed axis, so it neither reads the halo nor receives arrivals), 2 = boundary
__device__ __forceinline__ int dom_part(const int4& v, const SubParams& S)
{
    const int pc[3] = {v.y >> 1, v.z >> 1, v.w >> 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!S.dec[a]) continue;
        const int gcell = imodk(pc[a] + S.O[a], S.Gc[a]);
        const int lo = imodk((gcell / S.D[a]) * S.D[a] - S.O[a], S.Gc[a]);   // the domain's first local cell
        if (lo < 3 || lo + S.D[a] + 3 > S.Lb[a]) return 2;
    }
    return 1;
}

__device__ __forceinline__ void reset_phase_counters(DevCounters* ctr)
{
    ctr->nseg = 0; ctr->total = 0; ctr->nrun = 0; ctr->nrows = 0; ctr->chunk = 0; ctr->nhot = 0; ctr->ncold = 0;
    ctr->nseg2 = 0; ctr->chunk2 = 0; ctr->bready = 0; ctr->nexit = 0; ctr->nbdom = 0;
}
// the boundary segments of phase ph are complete: release them to the running engine
static __global__ void publish_boundary_kernel(DevCounters* ctr, const PhaseInfo* __restrict__ ph)
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctr->t_pub = t;
    __threadfence();
    asm volatile("st.release.gpu.global.s64 [%0], %1;" :: "l"(&ctr->bready), "l"(ph->phase + 1) : "memory");
}

// nvac = slot capacity; nvac_dev (multi-rank) = live slot count (slots may be departed: vac.x < 0);
// part 0: every domain (and the counters are reset here), 1: interior domains only, 2: boundary domains only
static __global__ void activate_kernel(const int4* __restrict__ vac, int nvac, const int* __restrict__ nvac_dev, SubParams S,
                                const PhaseInfo* __restrict__ ph, int* dmin, int* head, int* next, DevCounters* ctr,
                                int part = 0, long long* bdom = nullptr)
{
    // (programmatic dependent launch: this grid may be resident before the previous kernel has finished; it reads
    // nothing before the wait, and lets the segments kernel after it launch at once)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0 && part == 0) reset_phase_counters(ctr);
    const int n = nvac_dev ? min(*nvac_dev, nvac) : nvac;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 v = vac[i];
        if (v.x < 0) continue;
        long long d; int sec;
        dom_sector(v, S, d, sec);
        if (sec != ph->sector) continue;
        if (part != 0 && dom_part(v, S) != part) continue;
        atomicMin(&dmin[d], S.gid ? S.gid[i] : i);       // owner = smallest global slot id
        const int prev = atomicExch(&head[d], i);
        next[i] = prev;
        // (overlap) the first member of a boundary domain lists the domain for segments_boundary_kernel
        if (bdom && prev < 0 && dom_part(v, S) == 2) bdom[atomicAdd(&ctr->nbdom, 1ull)] = d;
    }
}

// Block-aggregated allocation: one atomic per block, offsets in thread (= slot) order inside the
// block, so consecutive segments/rows are spatially close (slots are numbered in site order) and a
// 128-row tile of the barrier kernel touches few lattice pages.  Returns this thread's exclusive
// offset; `total` receives the block sum.  blockDim.x must be 256.
__device__ __forceinline__ int block_alloc(int v, unsigned long long* counter)
{
    __shared__ int wsum[8];
    __shared__ int base_s;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) { const int t = wsum[w]; wsum[w] = tot; tot += t; }
        base_s = tot ? (int)atomicAdd(counter, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    const int r = base_s + wsum[wid] + incl - v;
    __syncthreads();
    return r;
}

__device__ __forceinline__ void segments_one(int i, int n, const int4* __restrict__ vac, const SubParams& S,
                                             const PhaseInfo* __restrict__ ph, int* dmin, int* head,
                                             const int* __restrict__ next, Segment* segs, int* members,
                                             uint8_t* mactive, DevCounters* ctr, int4* mpos,
                                             const unsigned char* memo, int seg_cap, double hot_events, int part,
                                             Segment* segs2)
{
    long long d = 0;
    int sec = -1;
    bool owner = false;
    int cnt = 0;
    if (i < n) {
        const int4 v = vac[i];
        if (v.x >= 0) {
            dom_sector(v, S, d, sec);
            owner = (sec == ph->sector && (part == 0 || dom_part(v, S) == part) &&
                     dmin[d] == (S.gid ? S.gid[i] : i));                        // smallest global slot owns
            if (owner)
                for (int j = head[d]; j >= 0; j = next[j]) ++cnt;
        }
    }
    const int off = block_alloc(cnt, &ctr->total);
    int seg;
    if (part == 2) {
        // boundary segments (multi-rank overlap): their own list, handed out after the interior ones
        seg = block_alloc(owner ? 1 : 0, &ctr->nseg2);
    } else if (memo) {
        // phase engine: order the segment list by expected events (processing order is free, R6).  A domain
        // whose last memoised rates predict >= hot_events events in the window (R_d * window) goes to the
        // front, the rest fill the list from the back; CTAs claim the front first, so long event chains
        // start at the first iteration instead of after a refill (shorter phase tail).
        double Rd = 0.0;
        if (owner)
            for (int j = head[d]; j >= 0; j = next[j]) {
                const double r = *reinterpret_cast<const double*>(memo + (size_t)(2 * j) * kMemoBytes + kMemoROff);
                if (r > 0.0) Rd += r;                    // empty entries (NaN) and dead vacancies add nothing
            }
        const bool hot = owner && Rd * S.window >= hot_events;
        const int h = block_alloc(hot ? 1 : 0, &ctr->nhot);
        const int k = block_alloc(owner && !hot ? 1 : 0, &ctr->ncold);
        seg = hot ? h : seg_cap - 1 - k;
        block_alloc(owner ? 1 : 0, &ctr->nseg);
    } else {
        seg = block_alloc(owner ? 1 : 0, &ctr->nseg);
    }
    if (!owner) return;
    int c = 0;
    for (int j = head[d]; j >= 0; j = next[j]) members[off + (c++)] = j;
    for (int a = 1; a < cnt; ++a) {                     // insertion sort by global slot id
        const int key = members[off + a];
        const int kg = S.gid ? S.gid[key] : key;
        int b = a - 1;
        while (b >= 0 && (S.gid ? S.gid[members[off + b]] : members[off + b]) > kg) {
            members[off + b + 1] = members[off + b];
            --b;
        }
        members[off + b + 1] = key;
    }
    for (int a = 0; a < cnt; ++a) mactive[off + a] = 1;
    if (mpos)
        for (int a = 0; a < cnt; ++a) mpos[off + a] = vac[members[off + a]];   // positions for the phase engine
    Segment sg;
    sg.dom = d; sg.off = off; sg.cnt = cnt; sg.t = 0.0; sg.it = 0u; sg.running = 1;
    (part == 2 ? segs2 : segs)[seg] = sg;
    head[d] = -1;
    dmin[d] = INT_MAX;
}


static __global__ void __launch_bounds__(256) segments_kernel(const int4* __restrict__ vac, int nvac,
                                                       const int* __restrict__ nvac_dev, SubParams S,
                                                       const PhaseInfo* __restrict__ ph, int* dmin, int* head,
                                                       const int* __restrict__ next, Segment* segs, int* members,
                                                       uint8_t* mactive, DevCounters* ctr, int4* mpos,
                                                       const unsigned char* memo = nullptr, int seg_cap = 0,
                                                       double hot_events = 0.0, int part = 0, Segment* segs2 = nullptr)
{
    // the phase engine launched after this kernel may start its prologue now (it waits for this grid's
    // completion with griddepcontrol.wait before it reads anything written here)
    asm volatile("griddepcontrol.wait;" ::: "memory");                 // (the activate kernel's lists)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int n = nvac_dev ? min(*nvac_dev, nvac) : nvac;
    // block-uniform trip count: block_alloc needs every thread of the block
    for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x)
        segments_one(i0 + (int)threadIdx.x, n, vac, S, ph, dmin, head, next, segs, members, mactive, ctr, mpos, memo,
                     seg_cap, hot_events, part, segs2);
}

// segments of the boundary domains of the phase (their lists were built by activate_kernel and by the arrivals of
// unpack_p2p_kernel, which also listed the domains in bdom): one thread per listed domain, block-uniform trip
// count for block_alloc
static __global__ void __launch_bounds__(256) segments_boundary_kernel(const long long* __restrict__ bdom, SubParams S,
                                                                      const int4* __restrict__ vac, int* dmin, int* head,
                                                                      const int* __restrict__ next, Segment* segs2,
                                                                      int* members, uint8_t* mactive, DevCounters* ctr,
                                                                      int4* mpos)
{
    const long long nb = (long long)*(volatile unsigned long long*)&ctr->nbdom;
    for (long long k0 = (long long)blockIdx.x * blockDim.x; k0 < nb; k0 += (long long)gridDim.x * blockDim.x) {
        const long long k = k0 + threadIdx.x;
        long long d = 0;
        int cnt = 0;
        if (k < nb) {
            d = bdom[k];
            for (int j = head[d]; j >= 0; j = next[j]) ++cnt;
        }
        const int off = block_alloc(cnt, &ctr->total);
        const int seg = block_alloc(cnt > 0 ? 1 : 0, &ctr->nseg2);
        if (cnt == 0) continue;
        int c = 0;
        for (int j = head[d]; j >= 0; j = next[j]) members[off + (c++)] = j;
        for (int a = 1; a < cnt; ++a) {                 // insertion sort by global slot id
            const int key = members[off + a];
            const int kg = S.gid[key];
            int b = a - 1;
            while (b >= 0 && S.gid[members[off + b]] > kg) {
                members[off + b + 1] = members[off + b];
                --b;
            }
            members[off + b + 1] = key;
        }
        for (int a = 0; a < cnt; ++a) { mactive[off + a] = 1; mpos[off + a] = vac[members[off + a]]; }
        Segment sg;
        sg.dom = d; sg.off = off; sg.cnt = cnt; sg.t = 0.0; sg.it = 0u; sg.running = 1;
        segs2[seg] = sg;
        head[d] = -1;
        dmin[d] = INT_MAX;
    }
}

// rows of this inner iteration = active members of running segments; also resets nrun
static __global__ void __launch_bounds__(256) rows_kernel(const Segment* __restrict__ segs, const int* __restrict__ members,
                                                   const uint8_t* __restrict__ mactive, int* rows, DevCounters* ctr)
{
    const int nseg = (int)ctr->nseg;
    for (int s0 = blockIdx.x * blockDim.x; s0 < nseg; s0 += gridDim.x * blockDim.x) {   // block-uniform loop
        const int s = s0 + threadIdx.x;
        Segment sg;
        int m = 0;
        if (s < nseg) {
            sg = segs[s];
            if (sg.running)
                for (int a = 0; a < sg.cnt; ++a) m += mactive[sg.off + a] ? 1 : 0;
        }
        int r = block_alloc(m, &ctr->nrows);
        if (m)
            for (int a = 0; a < sg.cnt; ++a)
                if (mactive[sg.off + a]) rows[r++] = members[sg.off + a];
    }
}

static __global__ void select_sub_kernel(uint8_t* species, int4* vac, Frame F, GeomTables G, SubParams S,
                                  const PhaseInfo* __restrict__ ph, Segment* segs, const int* __restrict__ members,
                                  uint8_t* mactive, const double* __restrict__ rates, const double* __restrict__ Rsum,
                                  double* scratch, int* iscratch, DevCounters* ctr)
{
    const int nseg = (int)ctr->nseg;
    const int sector = ph->sector;
    const unsigned long long p = (unsigned long long)ph->phase;
    unsigned long long evals = 0, events = 0;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += gridDim.x * blockDim.x) {
        Segment sg = segs[s];
        if (!sg.running) continue;
        double lbuf[32];                               // small competing sets: tree in registers/L1
        int lidx[16];
        const bool small = sg.cnt <= 16;
        double* buf = small ? lbuf : scratch + 4 * (size_t)sg.off;   // disjoint per segment: 2P-1 <= 4*cnt
        int* idx = small ? lidx : iscratch + sg.off;
        int m = 0;
        for (int a = 0; a < sg.cnt; ++a)
            if (mactive[sg.off + a]) {
                buf[m] = Rsum[members[sg.off + a]];
                idx[m] = a;
                ++m;
            }
        bool stop = false;
        if (m == 0) {
            stop = true;
        } else {
            evals += 8ull * (unsigned long long)m;
            int P = 1, nlev = 0;
            const double Rd = tree_build(buf, m, P, nlev);
            if (!(Rd > 0.0)) {
                stop = true;
            } else {
                double u_sel, u_t;
                philox_uniforms(S.seed, make_uint4(sg.it, (uint32_t)sg.dom, (uint32_t)p, (uint32_t)(p >> 32)), u_sel, u_t);
                const double dt = __ddiv_rn(-det_log(u_t), Rd);
                if (__dadd_rn(sg.t, dt) > S.window) {
                    stop = true;                          // overshooting draw discarded
                } else {
                    double r = __dmul_rn(u_sel, Rd);
                    const int leaf = tree_descend(buf, m, P, nlev, r);
                    const int a = idx[leaf];
                    const int slot = members[sg.off + a];
                    const int k = pick_hop(rates + (size_t)slot * 8, r);
                    const int4 ov = vac[slot];
                    const int4 nv = apply_hop(species, vac, slot, k, F, G);
                    long long d2; int sec2;
                    dom_sector(nv, S, d2, sec2);
                    if (d2 != sg.dom || sec2 != sector) mactive[sg.off + a] = 0;
                    if (S.log) {
                        // multi-rank: log writes a neighbour rank must see, and departures from the block
                        if (near_face(F, ov.y, ov.z, ov.w))
                            log_entry(S.log, S.nlog, S.logcap, ov.y, ov.z, ov.w,
                                      species[site_of(F, ov.x, ov.y, ov.z, ov.w)]);
                        if (near_face(F, nv.y, nv.z, nv.w))
                            log_entry(S.log, S.nlog, S.logcap, nv.y, nv.z, nv.w, kVac);
                        bool out = false;
                        const int np[3] = {nv.y, nv.z, nv.w};
                        for (int ax = 0; ax < 3; ++ax)
                            if (!F.wrap[ax] && (np[ax] < 0 || np[ax] >= 2 * F.L[ax])) out = true;
                        if (out) {
                            log_entry(S.log, S.nlog, S.logcap, nv.y, nv.z, nv.w, kMigrateBase + S.gid[slot]);
                            depart_slot(vac, S, slot);          // departed: re-created by the owner rank
                        }
                    }
                    sg.t = __dadd_rn(sg.t, dt);
                    sg.it += 1u;
                    events += 1;
                }
            }
        }
        if (stop) sg.running = 0;
        segs[s] = sg;
    }
    if (evals) atomicAdd(&ctr->hop_evals, evals);
    if (events) {
        atomicAdd(&ctr->events, events);
        atomicAdd(&ctr->nrun, events);
    }
}

// a8: continue the inner loop while some domain applied an event; resets nrun/nrows for the next trip
static __global__ void loop_cond_kernel(DevCounters* ctr, cudaGraphConditionalHandle handle)
{
    const unsigned long long run = ctr->nrun;
    ctr->nrun = 0;
    ctr->nrows = 0;
    cudaGraphSetConditional(handle, run > 0 ? 1u : 0u);
}

static __global__ void add_window_kernel(double* clock, int nvox, double w)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < nvox) clock[v] = __dadd_rn(clock[v], w);
}

static __global__ void fill_int_kernel(int* p, long long n, int val)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = val;
}

// ------------------------------------------------------------------ a0: vacancy registry by device scan
// 16 sites per thread (one uint4), 4096 per block.  Pass 1 counts vacancies and the max species code
// per block; pass 2 (one block) scans the block counts; pass 3 writes positions in site order.
constexpr int kScanThreads = 256;
constexpr int kScanSites = kScanThreads * 16;

__device__ __forceinline__ int vac_in_word(uint32_t w)
{
    int c = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) c += ((w >> (8 * b)) & 0xFF) == kVac;
    return c;
}

static __global__ void scan_count_kernel(const uint4* __restrict__ sp, long long nwords, int* bcount, unsigned int* maxcode)
{
    const long long wi = (long long)blockIdx.x * kScanThreads + threadIdx.x;
    int c = 0;
    unsigned int mx = 0;
    if (wi < nwords) {
        const uint4 v = sp[wi];
        c = vac_in_word(v.x) + vac_in_word(v.y) + vac_in_word(v.z) + vac_in_word(v.w);
        const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < 4; ++b) mx = max(mx, (ws[q] >> (8 * b)) & 0xFFu);
    }
    __shared__ int sc[kScanThreads / 32];
    __shared__ unsigned int sm[kScanThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) { sc[threadIdx.x >> 5] = c; sm[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0; unsigned int m = 0;
        for (int i = 0; i < kScanThreads / 32; ++i) { t += sc[i]; m = max(m, sm[i]); }
        bcount[blockIdx.x] = t;
        if (m > kVac) atomicMax(maxcode, m);
    }
}

// exclusive scan of n ints in place (single block of 1024 threads); total -> *total
static __global__ void __launch_bounds__(1024) scan_blocks_kernel(int* a, int n, long long* total)
{
    __shared__ long long part[1024];
    const int per = (n + 1023) / 1024;
    const int b0 = threadIdx.x * per;
    long long s = 0;
    for (int i = b0; i < min(n, b0 + per); ++i) s += a[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long acc = 0;
        for (int i = 0; i < 1024; ++i) { const long long t = part[i]; part[i] = acc; acc += t; }
        *total = acc;
    }
    __syncthreads();
    long long acc = part[threadIdx.x];
    for (int i = b0; i < min(n, b0 + per); ++i) { const int t = a[i]; a[i] = (int)acc; acc += t; }
}

static __global__ void scan_write_kernel(const uint4* __restrict__ sp, long long nwords, const int* __restrict__ boff,
                                  Frame F, int4* vac)
{
    const long long wi = (long long)blockIdx.x * kScanThreads + threadIdx.x;
    uint4 v = make_uint4(0, 0, 0, 0);
    int c = 0;
    if (wi < nwords) {
        v = sp[wi];
        c = vac_in_word(v.x) + vac_in_word(v.y) + vac_in_word(v.z) + vac_in_word(v.w);
    }
    // block-exclusive prefix of per-thread counts (thread order == site order)
    __shared__ int wsum[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int wbase = 0;
    for (int i = 0; i < wid; ++i) wbase += wsum[i];
    if (c == 0) return;
    int pos = boff[blockIdx.x] + wbase + incl - c;
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
    const long long csites = 2ll * F.L[0] * F.L[1] * F.L[2];      // canonical sites per voxel
    for (int q = 0; q < 4; ++q)
        for (int b = 0; b < 4; ++b)
            if (((ws[q] >> (8 * b)) & 0xFF) == kVac) {
                const long long site = wi * 16 + q * 4 + b;
                const int vox = (int)(site / csites);
                const long long li = site - (long long)vox * csites;
                const int bb = (int)(li & 1);
                const long long cell = li >> 1;
                const int x = (int)(cell % F.L[0]);
                const int y = (int)((cell / F.L[0]) % F.L[1]);
                const int z = (int)(cell / ((long long)F.L[0] * F.L[1]));
                vac[pos++] = make_int4(vox, 2 * x + bb, 2 * y + bb, 2 * z + bb);
            }
}

// canonical (x fastest, basis interleaved) <-> storage (halo + ghosts) layout conversions, one 8-byte
// brick line (4 cells along x x 2 basis sites) per thread, 16 threads per 128-byte brick: every brick is
// written (scatter) or read (gather) by one half-warp as a whole L2 line.
__device__ __forceinline__ int wrap_axis(int c, int L, int wrap, bool& ok)
{
    if (c >= 0 && c < L) return c;
    if (!wrap) { ok = false; return 0; }
    return ((c % L) + L) % L;
}

// storage brick lines (including the halo) <- canonical; halo cells on periodic axes get the images, on
// decomposed axes zeros (filled later by the halo exchange)
static __global__ void scatter_storage_kernel(const uint8_t* __restrict__ canon, uint8_t* storage, Frame F, int nvox)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nbv = (long long)F.NB[0] * F.NB[1] * F.NB[2];
    if (t >= 16 * nbv * nvox) return;
    const long long brick = t >> 4;
    const int l = (int)(t & 15), ly = l & 3, lz = l >> 2;
    const int vox = (int)(brick / nbv);
    const long long bi = brick - (long long)vox * nbv;
    const int bx = (int)(bi % F.NB[0]), by = (int)((bi / F.NB[0]) % F.NB[1]), bz = (int)(bi / ((long long)F.NB[0] * F.NB[1]));
    bool ok = true;
    const int y = wrap_axis(4 * by + ly - kHalo, F.L[1], F.wrap[1], ok);
    const int z = wrap_axis(4 * bz + lz - kHalo, F.L[2], F.wrap[2], ok);
    const long long csites = 2ll * F.L[0] * F.L[1] * F.L[2];
    const uint8_t* row = canon + (long long)vox * csites + 2ll * F.L[0] * (y + (long long)F.L[1] * z);
    unsigned long long v = 0;
    if (ok) {
        const int x0 = 4 * bx - kHalo;
        if (x0 >= 0 && x0 + 3 < F.L[0]) {
            const uint32_t* r4 = reinterpret_cast<const uint32_t*>(row + 2 * x0);   // 2*x0 = 8bx - 4: 4-aligned
            v = (unsigned long long)__ldg(r4) | ((unsigned long long)__ldg(r4 + 1) << 32);
        } else {
            for (int q = 0; q < 4; ++q) {
                bool okx = true;
                const int x = wrap_axis(x0 + q, F.L[0], F.wrap[0], okx);
                if (okx) v |= ((unsigned long long)row[2 * x] | ((unsigned long long)row[2 * x + 1] << 8)) << (16 * q);
            }
        }
    }
    uint8_t* dst = storage + (long long)vox * F.sites + (brick - (long long)vox * nbv) * 128 + (((lz << 2) | ly) << 3);
    *reinterpret_cast<unsigned long long*>(dst) = v;
}

// canonical <- storage (owned cells only): 8 canonical bytes per thread from two half brick lines
static __global__ void gather_canonical_kernel(const uint8_t* __restrict__ storage, uint8_t* canon, Frame F, int nvox)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nx = (F.L[0] + 3) >> 2;
    const long long per_vox = (long long)nx * F.L[1] * F.L[2];
    if (t >= per_vox * nvox) return;
    const int vox = (int)(t / per_vox);
    const long long r = t - (long long)vox * per_vox;
    const int k = (int)(r % nx);
    const long long yz = r / nx;
    const int y = (int)(yz % F.L[1]), z = (int)(yz / F.L[1]);
    uint8_t* dst = canon + (long long)vox * 2ll * F.L[0] * F.L[1] * F.L[2] + 2ll * F.L[0] * (y + (long long)F.L[1] * z);
    const int x0 = 4 * k;
    if (x0 + 3 < F.L[0]) {
        // storage cells x0+2 .. x0+5: the upper half of brick line k and the lower half of line k+1
        const uint8_t* base = storage + site_of(F, vox, 2 * x0, 2 * y, 2 * z);           // (x0+2)&3 == 2: +4 bytes
        const uint32_t lo = *reinterpret_cast<const uint32_t*>(base);
        const uint32_t hi = *reinterpret_cast<const uint32_t*>(storage + site_of(F, vox, 2 * x0 + 4, 2 * y, 2 * z));
        const unsigned long long v = (unsigned long long)lo | ((unsigned long long)hi << 32);
        if ((reinterpret_cast<uintptr_t>(dst + 2 * x0) & 7) == 0) {
            *reinterpret_cast<unsigned long long*>(dst + 2 * x0) = v;
        } else {
            *reinterpret_cast<uint32_t*>(dst + 2 * x0) = lo;
            *reinterpret_cast<uint32_t*>(dst + 2 * x0 + 4) = hi;
        }
    } else {
        for (int x = x0; x < F.L[0]; ++x)
            for (int bb = 0; bb < 2; ++bb) dst[2 * x + bb] = storage[site_of(F, vox, 2 * x + bb, 2 * y + bb, 2 * z + bb)];
    }
}

// vstart[v] = first slot whose voxel >= v (slots are in site order, hence voxel-major)
static __global__ void vstart_kernel(const int4* __restrict__ vac, int nvac, int nvox, int* vstart)
{
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v > nvox) return;
    int lo = 0, hi = nvac;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (vac[mid].x < v) lo = mid + 1; else hi = mid;
    }
    vstart[v] = lo;
}

} // namespace akmc
