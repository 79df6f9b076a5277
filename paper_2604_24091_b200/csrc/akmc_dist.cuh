// akmc_dist.cuh -- multi-GPU spatial decomposition (C5): per-rank blocks with a kHalo-cell halo,
// boundary-write logging, delta pack/unpack for the per-phase NCCL exchange, vacancy migration, and
// dense slab pack/unpack for the initial shift (X -> Y -> Z) halo fill (sec. V.B.3).
//
// Why deltas suffice (reading A20): within a phase, active sectors are >= 4 cells apart
// globally, reads reach 2 cells and writes 1 cell beyond a sector, so no site read by one rank in a
// phase is written by another rank in the same phase; after the phase every rank sends the sites it
// wrote that lie in a peer's extended region (block + halo), and the vacancies that left its block.
#pragma once
#include "akmc_device.cuh"
#include "akmc_route.h"

namespace akmc {

constexpr int kMaxPeers = 26;
constexpr int kMigrateBase = 16;          // entry code >= kMigrateBase: vacancy arrival, gid = code - base

struct DistParams {
    int O[3];                             // block origin (global cells)
    int G[3];                             // global cells per axis
    int npeer;
    int peerO[kMaxPeers][3];              // peer block origins (global cells)
    int cap;                              // entries per peer buffer (excluding the header entry)
};

__device__ __forceinline__ int imod(int a, int m) { const int r = a % m; return r < 0 ? r + m : r; }

// is global cell gc (per axis) inside the extended region (block + halo) of the block at origin o?
__device__ __forceinline__ bool in_extended(const int gc[3], const int o[3], const Frame& F, const DistParams& D)
{
    for (int a = 0; a < 3; ++a) {
        if (F.wrap[a]) continue;
        const int d = imod(gc[a] - o[a] + kHalo, D.G[a]);
        if (d >= F.L[a] + 2 * kHalo) return false;
    }
    return true;
}

__device__ __forceinline__ bool in_block(const int gc[3], const int o[3], const Frame& F, const DistParams& D)
{
    for (int a = 0; a < 3; ++a) {
        if (F.wrap[a]) continue;
        const int d = imod(gc[a] - o[a], D.G[a]);
        if (d >= F.L[a]) return false;
    }
    return true;
}

// does a site at owned half-cell coords p need to be logged (near a non-wrap face or outside the block)?
__device__ __forceinline__ bool near_face(const Frame& F, int px, int py, int pz)
{
    const int p[3] = {px, py, pz};
    for (int a = 0; a < 3; ++a) {
        if (F.wrap[a]) continue;
        const int c = p[a] >> 1;
        if (c < kHalo || c >= F.L[a] - kHalo) return true;
    }
    return false;
}

__device__ __forceinline__ void log_entry(int4* log, unsigned long long* nlog, int cap, int px, int py, int pz, int code)
{
    const unsigned long long i = atomicAdd(nlog, 1ull);
    if (i < (unsigned long long)cap) log[i] = make_int4(px, py, pz, code);
}

// Local slot reuse (multi-rank): a departure pushes its slot on the free list (depart_slot, akmc_kernels.cuh);
// an arrival pops one (FreeList.cnt[1] counts the pops of this exchange against the count nfree0 at kernel
// start -- no departures happen during an unpack) and only appends a new slot when the list is empty, so the
// slot range stays bounded by the most vacancies the block ever held at once, not by the migrations so far.
// The last block of the unpack folds the pops into the count.  The per-vacancy memo of a reused slot is kept:
// its entries are keyed by the full 64-byte window and rates are a pure function of the window (R7).
struct FreeList {
    int* slots;        // [vcap]
    int* cnt;          // [0] free slots, [1] pops of the running exchange, [2] finished unpack blocks
};

__device__ __forceinline__ int arrival_slot(const FreeList& FL, int nfree0, int* nvac_local)
{
    const int k = atomicAdd(&FL.cnt[1], 1);
    return k < nfree0 ? FL.slots[nfree0 - 1 - k] : atomicAdd(nvac_local, 1);
}

// (ep: the peer-mailbox exchange's device epoch counter -- the last block records that exchange `epoch` is done)
__device__ __forceinline__ void unpack_done(const FreeList& FL, int nfree0, unsigned long long* ep = nullptr,
                                            unsigned long long epoch = 0)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&FL.cnt[2], 1) == (int)gridDim.x - 1) {
            const int pops = atomicExch(&FL.cnt[1], 0);
            FL.cnt[0] = max(0, nfree0 - pops);
            FL.cnt[2] = 0;
            if (ep) *ep = epoch;
            __threadfence();
        }
    }
}

// pack the phase's log into per-peer send buffers (header entry 0 = count); global half-cell coords
// A site may be written several times in one phase (a vacancy enters and leaves it), so species entries
// carry the site's FINAL value, read here after the phase: duplicates are identical and the receiver may
// apply entries in any order.
static __global__ void pack_deltas_kernel(const int4* __restrict__ log, const unsigned long long* nlog_p, int logcap, Frame F,
                                   DistParams D, const uint8_t* __restrict__ species, int4* sendbuf, int* overflow)
{
    const int n = (int)min((unsigned long long)logcap, *nlog_p);
    if (blockIdx.x == 0 && threadIdx.x == 0 && *nlog_p > (unsigned long long)logcap) atomicAdd(overflow, 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int4 e = log[i];
        if (e.w < kMigrateBase) e.w = species[site_of(F, 0, e.x, e.y, e.z)];
        const int p[3] = {e.x, e.y, e.z};
        int gc[3], gp[3];
        for (int a = 0; a < 3; ++a) {
            gc[a] = imod((p[a] >> 1) + D.O[a], D.G[a]);
            gp[a] = 2 * gc[a] + (p[a] & 1);
        }
        for (int r = 0; r < D.npeer; ++r) {
            const bool want = (e.w >= kMigrateBase) ? in_block(gc, D.peerO[r], F, D) : in_extended(gc, D.peerO[r], F, D);
            if (!want) continue;
            int4* buf = sendbuf + (size_t)r * (D.cap + 1);
            const int k = atomicAdd(&buf[0].x, 1);
            if (k < D.cap) buf[1 + k] = make_int4(gp[0], gp[1], gp[2], e.w);
            else atomicAdd(overflow, 1);
        }
    }
}

static __global__ void clear_headers_kernel(int4* sendbuf, int npeer, int cap, unsigned long long* nlog)
{
    const int r = threadIdx.x;
    if (r < npeer) sendbuf[(size_t)r * (cap + 1)] = make_int4(0, 0, 0, 0);
    if (r == 0) *nlog = 0;
}

// apply received entries: species writes into block/halo (with wrap-axis ghosts); vacancy arrivals
static __global__ void unpack_deltas_kernel(const int4* __restrict__ recvbuf, int npeer, Frame F, DistParams D, uint8_t* species,
                                     int4* vac, int* gid, int* nvac_local, int vcap, FreeList FL, int* overflow)
{
    const int nfree0 = *(volatile int*)&FL.cnt[0];
    for (int r = 0; r < npeer; ++r) {
        const int4* buf = recvbuf + (size_t)r * (D.cap + 1);
        const int cnt = min(buf[0].x, D.cap);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
            const int4 e = buf[1 + i];
            const int gp[3] = {e.x, e.y, e.z};
            int lp[3];
            bool ok = true;
            for (int a = 0; a < 3; ++a) {
                if (F.wrap[a]) { lp[a] = gp[a]; continue; }
                int d = imod(gp[a] - 2 * D.O[a], 2 * D.G[a]);
                if (d >= 2 * (F.L[a] + kHalo)) d -= 2 * D.G[a];
                lp[a] = d;
                if (d < -2 * kHalo || d >= 2 * (F.L[a] + kHalo)) ok = false;
            }
            if (!ok) { atomicAdd(overflow, 1); continue; }
            if (e.w >= kMigrateBase) {
                const int slot = arrival_slot(FL, nfree0, nvac_local);
                if (slot < vcap) {
                    vac[slot] = make_int4(0, lp[0], lp[1], lp[2]);
                    gid[slot] = e.w - kMigrateBase;
                } else {
                    atomicAdd(overflow, 1);
                }
            } else {
                write_site(species, F, 0, lp[0], lp[1], lp[2], (uint8_t)e.w);
            }
        }
    }
    unpack_done(FL, nfree0);
}

// ---------------------------------------------------------------- shift-staged per-phase exchange (AKMC_EXCHANGE=shift)
// The paper's shift communication applied to the sparse per-phase deltas: the phase's entries (global
// half-cell coordinates, final value or migration code) go through the decomposed axes in order; at stage a a
// holder forwards an entry to the neighbour(s) along a chosen by route::shift_send (akmc_route.h), and every
// receiver applies what concerns it and keeps the entry for the later stages.  2 messages per axis instead of one
// per distinct neighbour block (tests/test_route_cpu.py: same deliveries as the direct exchange).
struct ShiftGeom {
    int P[3];          // this rank's block coordinates
    int L[3];          // block cells
    int grid[3];       // gpu grid
};

static __global__ void shift_collect_kernel(const int4* __restrict__ log, const unsigned long long* nlog_p, int logcap, Frame F,
                                            DistParams D, const uint8_t* __restrict__ species, int4* list, int* nlist,
                                            int* overflow)
{
    const int n = (int)min((unsigned long long)logcap, *nlog_p);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *nlist = n;
        if (*nlog_p > (unsigned long long)logcap) atomicAdd(overflow, 1);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int4 e = log[i];
        if (e.w < kMigrateBase) e.w = species[site_of(F, 0, e.x, e.y, e.z)];   // the site's FINAL value
        const int p[3] = {e.x, e.y, e.z};
        int gp[3];
        for (int a = 0; a < 3; ++a) gp[a] = 2 * imod((p[a] >> 1) + D.O[a], D.G[a]) + (p[a] & 1);
        list[i] = make_int4(gp[0], gp[1], gp[2], e.w);
    }
}

static __global__ void shift_pack_kernel(const int4* __restrict__ list, const int* nlist, int axis, ShiftGeom SG,
                                         int4* sendbuf, int cap, int* overflow)
{
    const int n = *nlist;
    const int ndir = route::shift_dirs(SG.grid[axis]);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 e = list[i];
        const int g[3] = {e.x >> 1, e.y >> 1, e.z >> 1};
        const bool mig = e.w >= kMigrateBase;
        for (int k = 0; k < ndir; ++k) {
            if (!route::shift_send(g, SG.P, axis, k == 0 ? 1 : -1, SG.L, SG.grid, kHalo, mig)) continue;
            int4* buf = sendbuf + (size_t)k * (cap + 1);
            const int q = atomicAdd(&buf[0].x, 1);
            if (q < cap) buf[1 + q] = e;
            else atomicAdd(overflow, 1);
        }
    }
}

// apply a stage's arrivals (species writes inside the extended region, vacancies arriving in the block) and keep
// them for the later stages
static __global__ void shift_unpack_kernel(const int4* __restrict__ recvbuf, int ndir, int cap, Frame F, DistParams D,
                                           uint8_t* species, int4* vac, int* gid, int* nvac_local, int vcap, FreeList FL,
                                           int4* list, int* nlist, int listcap, bool keep, int* overflow)
{
    const int nfree0 = *(volatile int*)&FL.cnt[0];
    for (int k = 0; k < ndir; ++k) {
        const int4* buf = recvbuf + (size_t)k * (cap + 1);
        const int cnt = min(buf[0].x, cap);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
            const int4 e = buf[1 + i];
            const int gp[3] = {e.x, e.y, e.z};
            int lp[3];
            bool in_ext = true, in_blk = true;
            for (int a = 0; a < 3; ++a) {
                if (F.wrap[a]) { lp[a] = gp[a]; continue; }
                int d = imod(gp[a] - 2 * D.O[a], 2 * D.G[a]);
                if (d >= 2 * (F.L[a] + kHalo)) d -= 2 * D.G[a];
                lp[a] = d;
                if (d < -2 * kHalo || d >= 2 * (F.L[a] + kHalo)) in_ext = false;
                if (d < 0 || d >= 2 * F.L[a]) in_blk = false;
            }
            if (e.w >= kMigrateBase) {
                if (in_blk && in_ext) {
                    const int slot = arrival_slot(FL, nfree0, nvac_local);
                    if (slot < vcap) {
                        vac[slot] = make_int4(0, lp[0], lp[1], lp[2]);
                        gid[slot] = e.w - kMigrateBase;
                    } else {
                        atomicAdd(overflow, 1);
                    }
                }
            } else if (in_ext) {
                write_site(species, F, 0, lp[0], lp[1], lp[2], (uint8_t)e.w);
            }
            if (keep) {
                const int q = atomicAdd(nlist, 1);
                if (q < listcap) list[q] = e;
                else atomicAdd(overflow, 1);
            }
        }
    }
    unpack_done(FL, nfree0);
}

// dense slab of cells (storage <-> buffer) for the initial halo fill.  Range per axis [lo, hi) in owned
// cells (may extend into the halo); buffer order x fastest, basis interleaved.
struct SlabRange { int lo[3], hi[3]; };

static __global__ void pack_slab_kernel(const uint8_t* __restrict__ species, Frame F, SlabRange R, uint8_t* buf)
{
    const int nx = R.hi[0] - R.lo[0], ny = R.hi[1] - R.lo[1], nz = R.hi[2] - R.lo[2];
    const long long n = 2ll * nx * ny * nz;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(i & 1);
        const long long c = i >> 1;
        const int x = R.lo[0] + (int)(c % nx), y = R.lo[1] + (int)((c / nx) % ny), z = R.lo[2] + (int)(c / ((long long)nx * ny));
        buf[i] = species[site_of(F, 0, 2 * x + b, 2 * y + b, 2 * z + b)];
    }
}

static __global__ void unpack_slab_kernel(const uint8_t* __restrict__ buf, Frame F, SlabRange R, uint8_t* species)
{
    const int nx = R.hi[0] - R.lo[0], ny = R.hi[1] - R.lo[1], nz = R.hi[2] - R.lo[2];
    const long long n = 2ll * nx * ny * nz;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(i & 1);
        const long long c = i >> 1;
        const int x = R.lo[0] + (int)(c % nx), y = R.lo[1] + (int)((c / nx) % ny), z = R.lo[2] + (int)(c / ((long long)nx * ny));
        write_site(species, F, 0, 2 * x + b, 2 * y + b, 2 * z + b, buf[i]);
    }
}

} // namespace akmc
