// akmc_api.cu -- C-ABI (include/akmc.h) of the B200 AKMC hot path: handle, validation, host
// loops of the serial (a10) and windowed-sublattice (a1-a9, reading A19) modes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <thread>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../../include/akmc.h"
#include "akmc_kernels.cuh"
#include "akmc_p2p.cuh"
#include "akmc_engine.cuh"
#include "akmc_world.cuh"
#include <nccl.h>

using namespace akmc;


// Device memory of a handle comes from the device's default stream-ordered pool with an unlimited release
// threshold: what akmc_free returns stays reserved in the process, so the next handle (a restart, bench.py's e2e
// handle) reuses it instead of paying the driver's fresh mapping of gigabytes again.  (The IPC-shared mailboxes of
// the multi-GPU exchange keep cudaMalloc: pool memory is not exportable through cudaIpcGetMemHandle.)
template <typename T>
static cudaError_t pool_malloc(T** p, size_t n)
{
    *p = nullptr;
    if (n == 0) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&pool, dev);
    if (e == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    void* q = nullptr;
    if (e == cudaSuccess) e = cudaMallocAsync(&q, n, (cudaStream_t)0);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)0);   // usable from any stream from here on
    if (e == cudaSuccess) *p = static_cast<T*>(q);
    return e;
}

#ifndef AKMC_PDL_LISTS
#define AKMC_PDL_LISTS 1        // activate / segments kernels with programmatic dependent launch (A/B knob)
#endif
// a launch with programmatic stream serialisation (the kernel waits with griddepcontrol.wait before it reads what
// the previous kernel writes; its blocks may be resident earlier and start without the launch gap)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args&&... args)
{
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = AKMC_PDL_LISTS;
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(block, 1, 1);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}


namespace {

thread_local std::string g_init_error;
constexpr int kDiagWords = 128 + 512 + 64 + 16;   // AKMC_PHASE_TIMING: sums, engine sums, iteration trace, bulk roles

// ------------------------------------------------------------------ host geometry (independent of the oracle)
// window: bcc vectors within 6.0 A at a0 = 2.866 A, sorted by (|h|^2, hx, hy, hz)  (A3, A4)
bool build_geometry(GeomTables& G)
{
    struct O { int h2, x, y, z; };
    std::vector<O> v;
    const double half_a0 = 2.866 / 2.0, rc = 6.0;
    for (int x = -5; x <= 5; ++x)
        for (int y = -5; y <= 5; ++y)
            for (int z = -5; z <= 5; ++z) {
                if (((x & 1) != (y & 1)) || ((y & 1) != (z & 1))) continue;
                if (x == 0 && y == 0 && z == 0) continue;
                const int h2 = x * x + y * y + z * z;
                if ((double)h2 * half_a0 * half_a0 <= rc * rc) v.push_back({h2, x, y, z});
            }
    std::sort(v.begin(), v.end(), [](const O& a, const O& b) {
        if (a.h2 != b.h2) return a.h2 < b.h2;
        if (a.x != b.x) return a.x < b.x;
        if (a.y != b.y) return a.y < b.y;
        return a.z < b.z;
    });
    if ((int)v.size() != kWin) return false;
    for (int j = 0; j < kWin; ++j) {
        G.off[j][0] = (int8_t)v[j].x; G.off[j][1] = (int8_t)v[j].y;
        G.off[j][2] = (int8_t)v[j].z; G.off[j][3] = (int8_t)v[j].h2;
    }
    auto slot_of = [&](int x, int y, int z) -> int {
        for (int j = 0; j < kWin; ++j)
            if (G.off[j][0] == x && G.off[j][1] == y && G.off[j][2] == z) return j;
        return -1;
    };
    // pair-KRA count lists per hop k: vacancy-side shells 1,2 without n_k (+1),
    // target-side shells 1,2 without the vacancy (-1); all inside the window (A.1)
    const int nn1[8][3] = {{-1,-1,-1},{-1,-1,1},{-1,1,-1},{-1,1,1},{1,-1,-1},{1,-1,1},{1,1,-1},{1,1,1}};
    const int nn2[6][3] = {{-2,0,0},{2,0,0},{0,-2,0},{0,2,0},{0,0,-2},{0,0,2}};
    for (int k = 0; k < kHops; ++k) {
        const int ex = G.off[k][0], ey = G.off[k][1], ez = G.off[k][2];
        int t = 0;
        for (int sh = 0; sh < 2; ++sh) {
            const int cnt = sh == 0 ? 8 : 6;
            for (int i = 0; i < cnt; ++i) {
                const int* d = sh == 0 ? nn1[i] : nn2[i];
                if (!(d[0] == ex && d[1] == ey && d[2] == ez)) {          // vacancy side, skip n_k
                    const int s = slot_of(d[0], d[1], d[2]);
                    if (s < 0) return false;
                    G.pair_slot[k][t] = (int8_t)s; G.pair_shell[k][t] = (int8_t)sh; G.pair_sign[k][t] = 1; ++t;
                }
                const int x = ex + d[0], y = ey + d[1], z = ez + d[2];
                if (!(x == 0 && y == 0 && z == 0)) {                        // target side, skip vacancy
                    const int s = slot_of(x, y, z);
                    if (s < 0) return false;
                    G.pair_slot[k][t] = (int8_t)s; G.pair_shell[k][t] = (int8_t)sh; G.pair_sign[k][t] = -1; ++t;
                }
            }
        }
        if (t != kPairTerms) return false;
    }
    return true;
}

// host Philox4x32-10 for the per-sweep sector permutation (A16/A19)
void philox_host(uint32_t c[4], uint32_t k0, uint32_t k1)
{
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[0] = n0; c[1] = (uint32_t)p1; c[2] = n2; c[3] = (uint32_t)p0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
}

void sector_permutation(uint64_t seed, int64_t sweep, int perm[8])
{
    uint32_t y[8];
    for (int j = 0; j < 2; ++j) {
        uint32_t c[4] = {(uint32_t)j, 0xFFFFFFFFu, (uint32_t)sweep, (uint32_t)((uint64_t)sweep >> 32)};
        philox_host(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        for (int i = 0; i < 4; ++i) y[4 * j + i] = c[i];
    }
    for (int i = 0; i < 8; ++i) perm[i] = i;
    for (int i = 7; i >= 1; --i) {
        const int j = (int)(y[i] % (uint32_t)(i + 1));
        std::swap(perm[i], perm[j]);
    }
}

} // namespace

struct akmc_handle {
    akmc_config cfg{};
    int dev = 0;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    bool sub = false;
    Frame F{};
    GeomTables G{};
    PhysParams P{};
    SubParams S{};
    int nvox = 0;
    int64_t nvac = 0, sites = 0;      // sites = canonical sites (all voxels)
    int64_t csites = 0, ssites = 0;   // canonical sites per voxel, storage sites (all voxels, with halos)
    long long ndom_total = 0;
    uint8_t* d_species = nullptr;
    int4* d_vac = nullptr;
    double *d_rates = nullptr, *d_R = nullptr, *d_E = nullptr, *d_scratch = nullptr;
    int* d_iscratch = nullptr;
    int* d_vstart = nullptr;
    double* d_clock = nullptr;
    long long* d_nev = nullptr;
    int* d_term = nullptr;
    int *d_dmin = nullptr, *d_head = nullptr, *d_next = nullptr, *d_members = nullptr, *d_rows = nullptr;
    int4* d_mpos = nullptr;           // member positions (phase engine)
    Segment* d_segs = nullptr;
    // multi-rank overlap of the per-phase exchange with the next phase's interior domains (step_sublattice_overlap)
    Segment* d_segs2 = nullptr;       // boundary domains' segments
    long long* d_bdom = nullptr;      // boundary domains holding active vacancies of the phase
    cudaStream_t side = nullptr;      // the exchange's receive side + the boundary activation
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool overlap_ok = false;          // p2p transport, phase engine: the overlapped sweep is available
    bool xpending = false;            // a packed exchange whose unpack has not been enqueued yet

    uint8_t* d_mactive = nullptr;
    DevCounters* d_ctr = nullptr;
    DevCounters* h_ctr = nullptr;     // pinned
    double* d_mlp = nullptr;
    float* d_b2 = nullptr;
    double* d_b3 = nullptr;
    float s2u = 1.0f, h1s = 1.0f;
    int act_shift = 0;                // t1: h1 scale 2^-t1 (prepare_engine_weights)
    double* d_W3d = nullptr;          // [256][8] FP64 W3 (layer 3 on CUDA cores)
    uint8_t* d_W2full = nullptr;      // bulk evaluator: W2^T images, N = 256 per K-step
    std::vector<double> W3h, b3h;     // host copies for the bulk evaluator's constant-bank parameters
    std::vector<float> b2h;
    bool bulk = true;                 // FP32 batches through the bulk evaluator (AKMC_EVAL_ENGINE=1: cluster evaluator)
    bool have_pair = false;           // eps / E0 given at init (pair tables valid)
    // dataflow sweep (f1; akmc_set_dataflow; akmc_engine.cu): one engine launch per sweep, tile readiness
    bool df = false;
    int df_tdom[3] = {1, 1, 1}, df_NT[3] = {1, 1, 1}, df_ntiles = 0, df_ring_cap = 8192, df_grid = 0;
    long long* d_done_phase = nullptr;
    int *d_tile_off = nullptr, *d_tile_cnt = nullptr, *d_tile_cur = nullptr, *d_tile_mem = nullptr;
    int *d_arr_cnt = nullptr, *d_arr_slot = nullptr, *d_ring_slot = nullptr, *d_df_iscratch = nullptr, *d_df_err = nullptr;
    int4* d_ring_pos = nullptr;
    unsigned long long* d_ring_key = nullptr;
    double* d_df_scratch = nullptr;
    // dynamic voxel scheduling (Eq. 10): per-voxel species counts and the segment dispatch order
    std::vector<unsigned long long> comp;   // [nvox][8]
    std::vector<int> vorder;                // voxel ids in dispatch order (descending W_v, stable)
    std::vector<double> vT;                 // per-voxel temperature (K)
    std::vector<int> vstart_host;           // [nvox + 1] slot ranges per voxel
    // world-model time mode (akmc_set_world_model; akmc_world.cu)
    bool world = false;
    double* d_tnet = nullptr;
    int world_H = 0;
    double world_tau = 1.0;
    unsigned long long* d_overflow = nullptr;
    // phase engine (akmc_engine.cuh)
    bool engine = true;               // false: legacy grid-synchronous inner loop (AKMC_LEGACY_LOOP=1)
    bool tc = false;                  // MLP at FP32 precision: cluster tensor-core evaluator
    bool serial_engine = false;       // serial / voxel-batch mode runs through the engine (voxel = domain)
    int n_clusters = 0;
    MemoEntry* d_memo = nullptr;      // [vcap][2]
    double* d_kT = nullptr;           // [n_voxels] kB * T_v (per-voxel temperature, C4 variant)
    double hot_events = 0.0;          // phase engine: domains expecting >= this many events go first (0: off;
                                      // A/B on C5: no change, profiles/r01_engine_timing.md)
    float* d_W1f = nullptr;           // [385][256]
    uint8_t* d_W2e = nullptr;         // [8][32 KiB]
    unsigned int* d_cursor = nullptr;
    uint8_t* d_stage = nullptr;       // [clusters][8][16 KiB] L2 staging of h1 rows (multicast)
    uint8_t* d_canon = nullptr;       // canonical-order lattice for akmc_state readbacks (lazy)
    uint8_t* d_wstore = nullptr;      // engine: per-CTA window scratch
    int* h_watch = nullptr;           // AKMC_WATCHDOG: engine progress words (mapped host memory)
    int* d_watch = nullptr;
    int profile = 0;
    std::vector<cudaEvent_t> ev;      // pairs
    size_t ev_used = 0;
    std::vector<cudaEvent_t> xev;     // AKMC_PHASE_TIMING, multi-rank host-stepped sweeps: (pack start, unpack start,
    size_t xev_used = 0;              // unpack end) triples around every exchange
    double xchg_ms[2] = {0.0, 0.0};   // summed pack / unpack (incl. the wait for the peers) ms
    int64_t xchg_n = 0;
    cudaEvent_t* xchg_mark = nullptr; // the current triple (exchange_deltas records the middle event)
    akmc_counters total{};
    int64_t sweep = 0;
    std::string err;
    int num_sms = 148;
    // per-sweep graph (sublattice mode): 8 phases, each with a conditional WHILE inner loop
    PhaseInfo* d_phase = nullptr;
    PhaseInfo* h_phase = nullptr;     // pinned
    cudaGraphExec_t sweep_exec = nullptr;
    cudaStream_t graph_stream = nullptr;   // stream the graph was instantiated for
    int graph_launches_per_sweep = 0;
    unsigned long long* d_phase_cycles = nullptr;   // AKMC_PHASE_TIMING diagnostics (kDiagWords)
    int vcap = 1;                     // vacancy slot capacity (multi-rank: arrivals append)
    // multi-rank spatial decomposition (C5); see akmc_dist.cuh
    bool multi = false;
    ncclComm_t comm = nullptr;
    int rc[3] = {0, 0, 0};            // this rank's block coordinates
    DistParams DP{};
    int peer_rank[kMaxPeers] = {};
    int* d_free = nullptr;            // free local slots (departures), reused by arrivals
    int* d_fcnt = nullptr;            // [0] free count [1] pops [2] unpack blocks done
    int* d_gid = nullptr;             // global slot id per local slot
    int* d_nvac = nullptr;            // live local slot count (device)
    int4* d_log = nullptr;
    unsigned long long* d_nlog = nullptr;
    int4 *d_send = nullptr, *d_recv = nullptr;
    int* d_dist_overflow = nullptr;
    cudaGraphExec_t phase_exec[8] = {};
    int64_t exchanges = 0, exchange_bytes = 0;
    // per-phase exchange over NVLink peer memory (CUDA IPC mailboxes; AKMC_EXCHANGE=nccl selects NCCL p2p)
    bool p2p = false;
    bool shift = false;                        // AKMC_EXCHANGE=shift: shift-staged NCCL exchange
    int4* d_slist = nullptr;                   // shift: entries of the phase (own + received)
    int* d_nslist = nullptr;
    int slistcap = 0;
    int64_t messages = 0;                      // per-phase messages sent (all phases)
    int4* d_mbox = nullptr;                    // [npeer][2][cap + 1]
    unsigned long long* d_mflag = nullptr;     // [kMaxPeers]
    int* d_pcnt = nullptr;
    unsigned long long* d_pepoch = nullptr;   // peer-mailbox exchanges completed (device-side epoch)
    unsigned int* d_pdone = nullptr;
    PeerBoxes PB{};
    void* ipc_box[kMaxPeers] = {};
    void* ipc_flag[kMaxPeers] = {};
};

namespace {

// per-voxel species counts of the canonical upload (composition is conserved per voxel in serial mode: vacancies
// never leave their voxel) -> the workload proxy's effective barrier (Eq. 10)
__global__ void voxel_comp_kernel(const uint8_t* __restrict__ canon, long long csites, unsigned long long* comp)
{
    __shared__ unsigned int cnt[8];
    if (threadIdx.x < 8) cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int v = blockIdx.y;
    const uint4* p = reinterpret_cast<const uint4*>(canon + (long long)v * csites);
    const long long nw = csites / 16;
    unsigned int loc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nw; i += (long long)gridDim.x * blockDim.x) {
        const uint4 w = p[i];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int b = 0; b < 4; ++b) loc[(ws[j] >> (8 * b)) & 7u] += 1u;
    }
    for (int s = 0; s < 8; ++s)
        if (loc[s]) atomicAdd(&cnt[s], loc[s]);
    __syncthreads();
    if (threadIdx.x < 8 && cnt[threadIdx.x]) atomicAdd(&comp[(size_t)v * 8 + threadIdx.x], (unsigned long long)cnt[threadIdx.x]);
}

int fail(akmc_handle* h, int code, const std::string& msg)
{
    if (h) h->err = msg; else g_init_error = msg;
    return code;
}

#define CK(h, x)                                                                                            \
    do {                                                                                                    \
        cudaError_t e_ = (x);                                                                               \
        if (e_ != cudaSuccess) return fail(h, AKMC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NCK(h, x)                                                                                           \
    do {                                                                                                    \
        ncclResult_t r_ = (x);                                                                              \
        if (r_ != ncclSuccess) return fail(h, AKMC_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

inline unsigned blocks_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

void free_all(akmc_handle* h)
{
    void* ptrs[] = {h->d_species, h->d_vac, h->d_rates, h->d_R, h->d_E, h->d_scratch, h->d_iscratch, h->d_vstart,
                    h->d_clock, h->d_nev, h->d_term, h->d_dmin, h->d_head, h->d_next, h->d_members, h->d_mpos, h->d_rows,
                    h->d_segs, h->d_mactive, h->d_ctr, h->d_mlp,
                    h->d_b2, h->d_b3, h->d_overflow, h->d_memo, h->d_W1f, h->d_W2e, h->d_W3d, h->d_W2full, h->d_tnet, h->d_cursor,
                    h->d_stage, h->d_canon, h->d_wstore, h->d_kT};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->d_phase) cudaFree(h->d_phase);
    if (h->h_phase) cudaFreeHost(h->h_phase);
    if (h->sweep_exec) cudaGraphExecDestroy(h->sweep_exec);
    if (h->h_ctr) cudaFreeHost(h->h_ctr);
    if (h->h_watch) cudaFreeHost(h->h_watch);
    for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : h->xev) cudaEventDestroy(e);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->d_segs2) cudaFree(h->d_segs2);
    if (h->d_bdom) cudaFree(h->d_bdom);
    for (int r = 0; r < kMaxPeers; ++r) {
        if (h->ipc_box[r]) cudaIpcCloseMemHandle(h->ipc_box[r]);
        if (h->ipc_flag[r]) cudaIpcCloseMemHandle(h->ipc_flag[r]);
    }
    void* dfptrs[] = {h->d_done_phase, h->d_tile_off, h->d_tile_cnt, h->d_tile_cur, h->d_tile_mem, h->d_arr_cnt,
                      h->d_arr_slot, h->d_ring_slot, h->d_df_iscratch, h->d_df_err, h->d_ring_pos, h->d_ring_key,
                      h->d_df_scratch};
    for (void* p : dfptrs)
        if (p) cudaFree(p);
    void* dptrs[] = {h->d_slist, h->d_nslist, h->d_free, h->d_fcnt, h->d_gid, h->d_nvac, h->d_log, h->d_nlog, h->d_send, h->d_recv, h->d_dist_overflow,
                     h->d_mbox, h->d_mflag, h->d_pcnt, h->d_pdone, h->d_pepoch};
    for (void* p : dptrs)
        if (p) cudaFree(p);
    for (int q = 0; q < 8; ++q)
        if (h->phase_exec[q]) cudaGraphExecDestroy(h->phase_exec[q]);
    if (h->comm) ncclCommDestroy(h->comm);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
}

int validate(const akmc_config* c, const double* eps, const double* E0, const double* mlp, std::string& why)
{
    for (int a = 0; a < 3; ++a) {
        if (c->cells[a] < 4 || (c->cells[a] & 1)) { why = "cells must be even and >= 4 (S:30)"; return AKMC_ERR_INVALID; }
        if (c->cells[a] > 4096) { why = "cells must be <= 4096 per axis (32-bit brick index)"; return AKMC_ERR_INVALID; }
    }
    if (c->n_voxels < 1) { why = "n_voxels must be >= 1"; return AKMC_ERR_INVALID; }
    if (c->n_species != kSpecies) { why = "n_species must be 7 (Fe Cu Ni Mn Si P V)"; return AKMC_ERR_INVALID; }
    if (!(c->temperature_K > 0.0) || !std::isfinite(c->temperature_K)) { why = "temperature must be > 0 (S:154)"; return AKMC_ERR_INVALID; }
    if (!(c->nu0 > 0.0) || !std::isfinite(c->nu0) || !(c->kB > 0.0) || !std::isfinite(c->kB)) { why = "nu0 and kB must be > 0"; return AKMC_ERR_INVALID; }
    if (c->barrier_model != AKMC_MODEL_PAIR && c->barrier_model != AKMC_MODEL_MLP) { why = "unknown barrier_model"; return AKMC_ERR_INVALID; }
    if (c->precision != AKMC_PREC_FP64 && c->precision != AKMC_PREC_FP32 && c->precision != AKMC_PREC_FP16_FAST) {
        why = "unknown precision"; return AKMC_ERR_INVALID;
    }
    const bool sub = c->domain_cells[0] || c->domain_cells[1] || c->domain_cells[2];
    if (sub) {
        for (int a = 0; a < 3; ++a) {
            const int D = c->domain_cells[a];
            if (D < 6 || (D & 1) || c->cells[a] % D) { why = "domain_cells must be even, >= 6 and divide cells (sector >= 3 cells, A20)"; return AKMC_ERR_INVALID; }
        }
        if (!(c->window_s > 0.0) || !std::isfinite(c->window_s)) { why = "window_s must be > 0 in sublattice mode"; return AKMC_ERR_INVALID; }
    }
    const int grid = c->gpu_grid[0] * c->gpu_grid[1] * c->gpu_grid[2];
    if (c->gpu_grid[0] < 1 || c->gpu_grid[1] < 1 || c->gpu_grid[2] < 1 || c->world != grid) { why = "world must equal prod(gpu_grid)"; return AKMC_ERR_INVALID; }
    if (c->rank < 0 || c->rank >= c->world) { why = "rank out of range"; return AKMC_ERR_INVALID; }
    if (c->world > 1) {
        if (!sub || c->n_voxels != 1) { why = "multi-rank decomposition needs sublattice mode and one voxel"; return AKMC_ERR_INVALID; }
        if (c->world > 4096) { why = "world too large"; return AKMC_ERR_INVALID; }
        for (int a = 0; a < 3; ++a)
            if (c->gpu_grid[a] > 1 && c->cells[a] < 2 * (kHalo + 2)) { why = "blocks too thin for the halo"; return AKMC_ERR_INVALID; }
    }
    if (c->barrier_model == AKMC_MODEL_PAIR) {
        if (!eps || !E0) { why = "pair model needs eps and E0"; return AKMC_ERR_INVALID; }
        for (int s = 0; s < 2; ++s)
            for (int a = 0; a < kSpecies; ++a)
                for (int b = 0; b < kSpecies; ++b) {
                    const double x = eps[(s * kSpecies + a) * kSpecies + b];
                    if (!std::isfinite(x)) { why = "non-finite eps"; return AKMC_ERR_INVALID; }
                    if (x != eps[(s * kSpecies + b) * kSpecies + a]) { why = "eps not symmetric (S:115)"; return AKMC_ERR_INVALID; }
                }
        for (int a = 0; a < kSpecies; ++a)
            if (!std::isfinite(E0[a])) { why = "non-finite E0"; return AKMC_ERR_INVALID; }
    } else {
        if (!mlp) { why = "MLP model needs weights"; return AKMC_ERR_INVALID; }
        const size_t n = 448 * kHid + kHid + kHid * kHid + kHid + kHid * 8 + 8;
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(mlp[i])) { why = "non-finite MLP weight"; return AKMC_ERR_INVALID; }
    }
    return AKMC_OK;
}

// FP32-equivalent evaluator weights: Fe-referenced layer-1 table, fp16 hi/lo UMMA images
// of the per-CTA W2 / W3 slices, and the power-of-two scales of weights and activations
int prepare_engine_weights(akmc_handle* h, const double* mlp)
{
    const double* W1 = mlp;
    const double* b1 = W1 + 448 * kHid;
    const double* W2 = b1 + kHid;
    const double* b2 = W2 + kHid * kHid;
    const double* W3 = b2 + kHid;
    const double* b3 = W3 + kHid * 8;
    constexpr double kLoScale = 2048.0;           // lo parts are stored * 2^11
    // power-of-two scale so that max|w| * 2^s <= 2^13 (fp16 hi/lo splits stay in range)
    auto scale_exp = [](const double* w, size_t n) {
        double mx = 0.0;
        for (size_t i = 0; i < n; ++i) mx = std::max(mx, std::fabs(w[i]));
        return mx > 0.0 ? 13 - (int)std::ceil(std::log2(mx)) : 0;
    };
    // layer 1, Fe-referenced (exact algebra, one species per slot): b1' = b1 + sum_slot W1[7*slot+Fe],
    // W1'(s, slot) = W1[7*slot+s] - W1[7*slot+Fe] for s = 1..6; table row 0 = b1', row 1+(s-1)*64+slot = W1'
    std::vector<double> w1p((size_t)kW1Rows * kHid);
    for (int j = 0; j < kHid; ++j) {
        double acc = b1[j];
        for (int s = 0; s < kWin; ++s) acc += W1[(size_t)(kSpecies * s + kFe) * kHid + j];
        w1p[j] = acc;
    }
    for (int s = 1; s < kSpecies; ++s)
        for (int slot = 0; slot < kWin; ++slot)
            for (int j = 0; j < kHid; ++j)
                w1p[(size_t)(1 + (s - 1) * kWin + slot) * kHid + j] =
                    W1[(size_t)(kSpecies * slot + s) * kHid + j] - W1[(size_t)(kSpecies * slot + kFe) * kHid + j];
    // activation bound over ALL windows: h1_j <= max(0, b1'_j + sum_slot max(0, max_s W1'(s,slot)_j)); the scale
    // 2^-t1 keeps every |h1| * 2^-t1 <= 2^15, so the fp16 hi part of an activation can never overflow (t1 = 0 for
    // O(1) activations: bits unchanged).  h2 is not split any more (layer 3 runs in FP64 on CUDA cores).
    double m1 = 0.0;
    for (int j = 0; j < kHid; ++j) {
        double u = w1p[j];
        for (int slot = 0; slot < kWin; ++slot) {
            double mx = 0.0;
            for (int s = 1; s < kSpecies; ++s) mx = std::max(mx, w1p[(size_t)(1 + (s - 1) * kWin + slot) * kHid + j]);
            u += mx;
        }
        m1 = std::max(m1, std::max(0.0, u));
    }
    // AKMC_NO_ACT_SCALE: fault injection for the overflow guard's test (no activation scaling)
    const bool no_scale = std::getenv("AKMC_NO_ACT_SCALE") != nullptr;
    const int t1 = (m1 > 32768.0 && !no_scale) ? (int)std::ceil(std::log2(m1 / 32768.0)) : 0;
    const int s2 = scale_exp(W2, (size_t)kHid * kHid);
    h->act_shift = t1;
    h->s2u = (float)std::ldexp(1.0, t1 - s2);
    h->h1s = (float)std::ldexp(1.0, -t1);
    std::vector<float> b2f(kHid);
    for (int i = 0; i < kHid; ++i) b2f[i] = (float)b2[i];
    h->W3h.assign(W3, W3 + (size_t)kHid * 8);
    h->b3h.assign(b3, b3 + 8);
    h->b2h = b2f;
    // per cluster CTA r: fp16 hi/lo UMMA images of W2^T columns [64r, 64r+64); W3 stays FP64
    {
        std::vector<float> w1f((size_t)kW1Rows * kHid);
        for (size_t i = 0; i < w1f.size(); ++i) w1f[i] = (float)w1p[i];
        const size_t w2b = (size_t)(kHid / 16) * 2 * kSliceN * 16 * 2;
        std::vector<uint8_t> w2e((size_t)kClusterN * w2b, 0);
        auto put_split = [&](uint8_t* stepbase, int N, int n, int kk, double w) {   // one K-step (16), hi then lo
            const __half hi = __float2half_rn((float)w);
            const __half lo = __float2half_rn((float)((w - (double)__half2float(hi)) * kLoScale));
            const size_t off = ((size_t)(kk / 8) * (N / 8) + n / 8) * 128 + (n % 8) * 16 + (kk % 8) * 2;
            const size_t split = (size_t)N * 16 * 2;
            reinterpret_cast<__half*>(stepbase + off)[0] = hi;
            reinterpret_cast<__half*>(stepbase + split + off)[0] = lo;
        };
        for (int r = 0; r < kClusterN; ++r)
            for (int k = 0; k < kHid; ++k)
                for (int c = 0; c < kSliceN; ++c)
                    put_split(w2e.data() + r * w2b + (size_t)(k / 16) * 2 * kSliceN * 16 * 2, kSliceN, c, k % 16,
                              std::ldexp(W2[(size_t)k * kHid + kSliceN * r + c], s2));
        // bulk evaluator: the whole W2^T per K-step (N = 256), [16][hi 8 KiB | lo 8 KiB]
        const size_t w2s = (size_t)kHid * 16 * 2 * 2;
        std::vector<uint8_t> w2f((size_t)(kHid / 16) * w2s, 0);
        for (int k = 0; k < kHid; ++k)
            for (int n = 0; n < kHid; ++n)
                put_split(w2f.data() + (size_t)(k / 16) * w2s, kHid, n, k % 16, std::ldexp(W2[(size_t)k * kHid + n], s2));
        CK(h, pool_malloc(&h->d_W2full, w2f.size()));
        CK(h, cudaMemcpy(h->d_W2full, w2f.data(), w2f.size(), cudaMemcpyHostToDevice));
        CK(h, pool_malloc(&h->d_W1f, w1f.size() * sizeof(float)));
        CK(h, pool_malloc(&h->d_W2e, w2e.size()));
        CK(h, pool_malloc(&h->d_W3d, (size_t)kHid * 8 * sizeof(double)));
        CK(h, cudaMemcpy(h->d_W1f, w1f.data(), w1f.size() * sizeof(float), cudaMemcpyHostToDevice));
        CK(h, cudaMemcpy(h->d_W2e, w2e.data(), w2e.size(), cudaMemcpyHostToDevice));
        CK(h, cudaMemcpy(h->d_W3d, W3, (size_t)kHid * 8 * sizeof(double), cudaMemcpyHostToDevice));
    }
    CK(h, pool_malloc(&h->d_b2, kHid * 4));
    CK(h, pool_malloc(&h->d_b3, 8 * 8));
    CK(h, cudaMemcpy(h->d_b2, b2f.data(), kHid * 4, cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(h->d_b3, b3, 8 * 8, cudaMemcpyHostToDevice));
    if (std::getenv("AKMC_PHASE_TIMING")) {
        CK(h, pool_malloc(&h->d_phase_cycles, kDiagWords * sizeof(unsigned long long)));
        CK(h, cudaMemset(h->d_phase_cycles, 0, kDiagWords * sizeof(unsigned long long)));
    }
    return AKMC_OK;
}

// Dynamic voxel scheduling (Eq. 10): W_v = M_v exp(-E_v / (kB T_v)) with M_v = 8 x the
// voxel's vacancies (feasible-event upper bound) and E_v = the composition-weighted mean base barrier E0 of its
// atoms (SPEC workload_proxy); voxels are dispatched in descending W_v (stable: ties keep voxel order), and the
// persistent engine's CTAs pull the next voxel from that list as soon as a slot frees (pull-on-finish).  The
// order changes no trajectory (voxels are independent, R6/R10) -- only the makespan of batches larger than the
// resident slots.
int order_voxels(akmc_handle* h)
{
    const int nv = h->nvox;
    std::vector<double> W((size_t)nv, 0.0);
    for (int v = 0; v < nv; ++v) {
        const int m = h->vstart_host[(size_t)v + 1] - h->vstart_host[(size_t)v];
        double e = 0.0, n = 0.0;
        for (int s = 0; s < kSpecies; ++s) {
            if (s == kVac) continue;
            const double c = (double)h->comp[(size_t)v * 8 + s];
            e += c * h->P.E0[s];
            n += c;
        }
        const double Ev = (n > 0.0 && h->have_pair) ? e / n : 0.0;
        W[(size_t)v] = 8.0 * m * std::exp(-Ev / (h->cfg.kB * h->vT[(size_t)v]));
    }
    h->vorder.resize((size_t)nv);
    for (int v = 0; v < nv; ++v) h->vorder[(size_t)v] = v;
    if (!std::getenv("AKMC_VOXEL_FIFO"))                  // A/B knob: FIFO (voxel id) dispatch
        std::stable_sort(h->vorder.begin(), h->vorder.end(), [&](int a, int b) { return W[(size_t)a] > W[(size_t)b]; });
    std::vector<Segment> sg((size_t)nv);
    for (int q = 0; q < nv; ++q) {
        const int v = h->vorder[(size_t)q];
        sg[(size_t)q] = Segment{(long long)v, h->vstart_host[(size_t)v], h->vstart_host[(size_t)v + 1] - h->vstart_host[(size_t)v],
                                0.0, 0u, 1};
    }
    CK(h, cudaMemcpy(h->d_segs, sg.data(), sg.size() * sizeof(Segment), cudaMemcpyHostToDevice));
    return AKMC_OK;
}

EngineParams engine_params(akmc_handle* h, int mode)
{
    EngineParams p{};
    p.mode = mode;
    p.model = h->cfg.barrier_model;
    p.species = h->d_species; p.vac = h->d_vac; p.F = h->F; p.G = h->G; p.P = h->P; p.S = h->S;
    p.S.seed = h->cfg.seed;                        // (serial handles leave the sublattice block unset)
    p.segs = h->d_segs; p.members = h->d_members; p.mpos = h->d_mpos; p.ctr = h->d_ctr; p.memo = h->d_memo;
    p.scratch = h->d_scratch; p.iscratch = h->d_iscratch; p.cursor = h->d_cursor;
    p.W.W1f = h->d_W1f; p.W.W2img = h->d_W2e; p.W.W3d = h->d_W3d; p.W.b2 = h->d_b2; p.W.b3 = h->d_b3;
    p.W.s2u = h->s2u; p.W.h1s = h->h1s; p.W.mlp64 = h->d_mlp;
    p.overflow = h->d_overflow;
    p.stage = h->d_stage;
    p.wstore = h->d_wstore;
    p.watch = h->d_watch;
    p.diag = h->d_phase_cycles ? h->d_phase_cycles + 32 : nullptr;
    p.seg_cap = (h->engine && h->hot_events > 0.0) ? h->vcap : 0;   // hot-first segment list (phase mode)
    p.fast = h->cfg.precision == AKMC_PREC_FP16_FAST ? 1 : 0;
    return p;
}

// evaluate rows -> rates/R/E with the handle's model at `prec`
int eval_rows(akmc_handle* h, const int* rows, const int* nrows_dev, int nrows_host, int max_rows,
              const uint8_t* windows, int prec, double* rates, double* R, double* E)
{
    if (max_rows <= 0) return AKMC_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->profile) {
        if (h->ev_used + 2 > h->ev.size()) {
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                CK(h, cudaEventCreate(&e));
                h->ev.push_back(e);
            }
        }
        e0 = h->ev[h->ev_used++];
        e1 = h->ev[h->ev_used++];
        CK(h, cudaEventRecord(e0, h->stream));
    }
    if (h->cfg.barrier_model == AKMC_MODEL_PAIR) {
        const unsigned grid = std::min<unsigned>(blocks_for(max_rows, 128), (unsigned)h->num_sms * 16u);
        eval_pair_kernel<<<grid, 128, 0, h->stream>>>(
            h->d_species, h->d_vac, windows, h->F, h->G, h->P, rows, nrows_dev, nrows_host, rates, R, E, h->d_ctr);
        CK(h, cudaGetLastError());
    } else if (prec == AKMC_PREC_FP64) {
        const unsigned grid = std::min<unsigned>((unsigned)max_rows, (unsigned)h->num_sms * 8u);
        eval_mlp_fp64_kernel<<<grid, 256, 0, h->stream>>>(h->d_species, h->d_vac, windows, h->F, h->G, h->P,
                                                           h->d_mlp, rows, nrows_dev, nrows_host, rates, R, E);
        CK(h, cudaGetLastError());
    } else if (h->bulk) {
        // FP32-equivalent / FP16-fast batches: the bulk evaluator (akmc_bulk.cu), row for row the phase engine's
        // arithmetic (akmc_eval.cuh) -- every path that produces a rate produces the same bits (R7)
        BulkParams p{};
        p.species = h->d_species; p.vac = h->d_vac; p.F = h->F; p.G = h->G; p.P = h->P;
        p.windows = windows; p.rows = rows; p.nrows_dev = nrows_dev; p.nrows_host = nrows_host;
        p.W = engine_params(h, kEngineEval).W;
        p.W2full = h->d_W2full;
        p.rates = rates; p.Rsum = R; p.E = E; p.overflow = h->d_overflow;
        p.fast = prec == AKMC_PREC_FP16_FAST ? 1 : 0;
        p.diag = h->d_phase_cycles ? h->d_phase_cycles + 128 + 512 + 64 : nullptr;   // last 16 diag words
        CK(h, launch_bulk(p, max_rows, h->num_sms, h->stream));
    } else {
        // the engine's cluster evaluator in eval mode (AKMC_EVAL_ENGINE=1; same arithmetic as the bulk evaluator)
        EngineParams p = engine_params(h, kEngineEval);
        p.windows = windows; p.rows = rows; p.nrows_dev = nrows_dev; p.nrows_host = nrows_host;
        p.rates = rates; p.Rsum = R; p.E = E;
        p.fast = prec == AKMC_PREC_FP16_FAST ? 1 : 0;
        CK(h, cudaMemsetAsync(h->d_cursor, 0, sizeof(unsigned int), h->stream));
        const int need = (max_rows + kRoundRows * kClusterN - 1) / (kRoundRows * kClusterN);
        CK(h, launch_engine(p, true, std::max(1, std::min(h->n_clusters, need)), h->num_sms, h->stream));
    }
    h->total.kernel_launches += 1;
    h->total.mlp_launches += 1;
    if (h->profile) CK(h, cudaEventRecord(e1, h->stream));
    return AKMC_OK;
}

int harvest_events(akmc_handle* h)
{
    if (!h->profile) return AKMC_OK;
    for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
        float ms = 0.f;
        CK(h, cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
        h->total.mlp_ms += ms;
    }
    h->ev_used = 0;
    for (size_t i = 0; i + 3 <= h->xev_used; i += 3) {
        float a = 0.f, b = 0.f;
        CK(h, cudaEventElapsedTime(&a, h->xev[i], h->xev[i + 1]));
        CK(h, cudaEventElapsedTime(&b, h->xev[i + 1], h->xev[i + 2]));
        h->xchg_ms[0] += a; h->xchg_ms[1] += b; h->xchg_n += 1;
    }
    h->xev_used = 0;
    return AKMC_OK;
}

// ------------------------------------------------------------------ multi-rank setup (C5)
int rank_of(const akmc_config& c, int x, int y, int z)
{
    const int gx = c.gpu_grid[0], gy = c.gpu_grid[1], gz = c.gpu_grid[2];
    x = ((x % gx) + gx) % gx; y = ((y % gy) + gy) % gy; z = ((z % gz) + gz) % gz;
    return x + gx * (y + gy * z);
}

// initial halo fill by shift communication X -> Y -> Z: along axis a the face slab spans the
// extended range of the axes already exchanged and the owned range of the later ones, so edges and
// corners propagate in 3 stages of 2 messages instead of 26 direct ones.
int halo_fill(akmc_handle* h)
{
    const akmc_config& c = h->cfg;
    for (int a = 0; a < 3; ++a) {
        if (h->F.wrap[a]) continue;
        SlabRange face_lo{}, face_hi{}, halo_lo{}, halo_hi{};
        long long cells = 1;
        for (int b = 0; b < 3; ++b) {
            int lo, hi;
            if (b < a) { lo = -kHalo; hi = c.cells[b] + kHalo; }
            else { lo = 0; hi = c.cells[b]; }
            face_lo.lo[b] = face_hi.lo[b] = halo_lo.lo[b] = halo_hi.lo[b] = lo;
            face_lo.hi[b] = face_hi.hi[b] = halo_lo.hi[b] = halo_hi.hi[b] = hi;
            if (b != a) cells *= (hi - lo);
        }
        face_lo.lo[a] = 0;                  face_lo.hi[a] = kHalo;
        face_hi.lo[a] = c.cells[a] - kHalo; face_hi.hi[a] = c.cells[a];
        halo_hi.lo[a] = c.cells[a];         halo_hi.hi[a] = c.cells[a] + kHalo;
        halo_lo.lo[a] = -kHalo;             halo_lo.hi[a] = 0;
        const size_t bytes = (size_t)(2 * kHalo * cells * 2);
        int e[3] = {0, 0, 0};
        e[a] = 1;
        const int minus = rank_of(c, h->rc[0] - e[0], h->rc[1] - e[1], h->rc[2] - e[2]);
        const int plus = rank_of(c, h->rc[0] + e[0], h->rc[1] + e[1], h->rc[2] + e[2]);
        uint8_t *sb = nullptr, *rb = nullptr;
        CK(h, pool_malloc(&sb, bytes));
        CK(h, pool_malloc(&rb, bytes));
        const unsigned grid = (unsigned)h->num_sms * 4u;
        // lower face -> minus neighbour's upper halo; upper face -> plus neighbour's lower halo
        pack_slab_kernel<<<grid, 256, 0, h->stream>>>(h->d_species, h->F, face_lo, sb);
        NCK(h, ncclGroupStart());
        NCK(h, ncclSend(sb, bytes, ncclChar, minus, h->comm, h->stream));
        NCK(h, ncclRecv(rb, bytes, ncclChar, plus, h->comm, h->stream));
        NCK(h, ncclGroupEnd());
        unpack_slab_kernel<<<grid, 256, 0, h->stream>>>(rb, h->F, halo_hi, h->d_species);
        pack_slab_kernel<<<grid, 256, 0, h->stream>>>(h->d_species, h->F, face_hi, sb);
        NCK(h, ncclGroupStart());
        NCK(h, ncclSend(sb, bytes, ncclChar, plus, h->comm, h->stream));
        NCK(h, ncclRecv(rb, bytes, ncclChar, minus, h->comm, h->stream));
        NCK(h, ncclGroupEnd());
        unpack_slab_kernel<<<grid, 256, 0, h->stream>>>(rb, h->F, halo_lo, h->d_species);
        CK(h, cudaStreamSynchronize(h->stream));
        cudaFree(sb);
        cudaFree(rb);
    }
    return AKMC_OK;
}

// distinct ranks at the 26 neighbour offsets along decomposed (non-wrap) axes of the block at grid coords rc
int peer_list(const akmc_config& c, const int rc[3], const int wrap[3], int* out)
{
    int np = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int d[3] = {dx, dy, dz};
                bool skip = dx == 0 && dy == 0 && dz == 0;
                for (int a = 0; a < 3; ++a)
                    if (wrap[a] && d[a] != 0) skip = true;
                if (skip) continue;
                const int r = rank_of(c, rc[0] + dx, rc[1] + dy, rc[2] + dz);
                if (r == rank_of(c, rc[0], rc[1], rc[2])) continue;
                bool seen = false;
                for (int i = 0; i < np; ++i) seen |= (out[i] == r);
                if (!seen) out[np++] = r;
            }
    return np;
}

// mailboxes for the per-phase exchange, mapped into every peer by CUDA IPC (handles all-gathered over NCCL)
int setup_p2p(akmc_handle* h)
{
    const akmc_config& c = h->cfg;
    const int np = h->DP.npeer;
    const size_t per = (size_t)(h->DP.cap + 1);
    CK(h, cudaMalloc(&h->d_mbox, std::max<size_t>(1, (size_t)np * 2 * per) * sizeof(int4)));
    CK(h, cudaMalloc(&h->d_mflag, kMaxPeers * sizeof(unsigned long long)));
    CK(h, pool_malloc(&h->d_pcnt, kMaxPeers * sizeof(int)));
    CK(h, pool_malloc(&h->d_pdone, sizeof(unsigned int)));
    CK(h, pool_malloc(&h->d_pepoch, sizeof(unsigned long long)));
    CK(h, cudaMemset(h->d_pepoch, 0, sizeof(unsigned long long)));
    CK(h, cudaMemset(h->d_mbox, 0, std::max<size_t>(1, (size_t)np * 2 * per) * sizeof(int4)));
    CK(h, cudaMemset(h->d_mflag, 0, kMaxPeers * sizeof(unsigned long long)));
    CK(h, cudaMemset(h->d_pcnt, 0, kMaxPeers * sizeof(int)));
    CK(h, cudaMemset(h->d_pdone, 0, sizeof(unsigned int)));
    cudaIpcMemHandle_t mine[2];
    CK(h, cudaIpcGetMemHandle(&mine[0], h->d_mbox));
    CK(h, cudaIpcGetMemHandle(&mine[1], h->d_mflag));
    const size_t hb = sizeof(mine);
    uint8_t *d_h = nullptr, *d_all = nullptr;
    CK(h, pool_malloc(&d_h, hb));
    CK(h, pool_malloc(&d_all, hb * c.world));
    CK(h, cudaMemcpy(d_h, mine, hb, cudaMemcpyHostToDevice));
    NCK(h, ncclAllGather(d_h, d_all, hb, ncclChar, h->comm, h->stream));
    std::vector<cudaIpcMemHandle_t> all((size_t)2 * c.world);
    CK(h, cudaMemcpyAsync(all.data(), d_all, hb * c.world, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    cudaFree(d_h);
    cudaFree(d_all);
    for (int r = 0; r < np; ++r) {
        const int pr = h->peer_rank[r];
        const int prc[3] = {pr % c.gpu_grid[0], (pr / c.gpu_grid[0]) % c.gpu_grid[1], pr / (c.gpu_grid[0] * c.gpu_grid[1])};
        int theirs[kMaxPeers];
        const int tn = peer_list(c, prc, h->F.wrap, theirs);
        int me = -1;
        for (int i = 0; i < tn; ++i)
            if (theirs[i] == c.rank) me = i;
        if (me < 0) return fail(h, AKMC_ERR_RUNTIME, "peer lists are not symmetric");
        CK(h, cudaIpcOpenMemHandle(&h->ipc_box[r], all[(size_t)2 * pr], cudaIpcMemLazyEnablePeerAccess));
        CK(h, cudaIpcOpenMemHandle(&h->ipc_flag[r], all[(size_t)2 * pr + 1], cudaIpcMemLazyEnablePeerAccess));
        h->PB.box[r] = reinterpret_cast<int4*>(h->ipc_box[r]) + (size_t)me * 2 * per;
        h->PB.flag[r] = reinterpret_cast<unsigned long long*>(h->ipc_flag[r]) + me;
    }
    h->PB.cnt = h->d_pcnt;
    h->PB.done = h->d_pdone;
    h->PB.ep = h->d_pepoch;
    h->p2p = true;
    return AKMC_OK;
}

int init_multi(akmc_handle* h)
{
    const akmc_config& c = h->cfg;
    ncclUniqueId id;
    static_assert(sizeof(ncclUniqueId) <= sizeof(c.nccl_id), "nccl id size");
    std::memcpy(&id, c.nccl_id, sizeof(id));
    const auto tv0 = std::chrono::steady_clock::now();
    NCK(h, ncclCommInitRank(&h->comm, c.world, id, c.rank));
    const auto tv1 = std::chrono::steady_clock::now();
    // peers: distinct ranks at the 26 neighbour offsets along decomposed (non-wrap) axes
    const int np = peer_list(c, h->rc, h->F.wrap, h->peer_rank);
    for (int i = 0; i < np; ++i) {
        const int r = h->peer_rank[i];
        h->DP.peerO[i][0] = (r % c.gpu_grid[0]) * c.cells[0];
        h->DP.peerO[i][1] = ((r / c.gpu_grid[0]) % c.gpu_grid[1]) * c.cells[1];
        h->DP.peerO[i][2] = (r / (c.gpu_grid[0] * c.gpu_grid[1])) * c.cells[2];
    }
    h->DP.npeer = np;
    h->DP.cap = 8192;
    h->S.logcap = 1 << 17;
    const size_t per = (size_t)(h->DP.cap + 1);
    CK(h, pool_malloc(&h->d_log, (size_t)h->S.logcap * sizeof(int4)));
    CK(h, pool_malloc(&h->d_nlog, sizeof(unsigned long long)));
    CK(h, pool_malloc(&h->d_send, std::max<size_t>(2, np) * per * sizeof(int4)));     // (shift: 2 buffers per axis)
    CK(h, pool_malloc(&h->d_recv, std::max<size_t>(2, np) * per * sizeof(int4)));
    CK(h, pool_malloc(&h->d_dist_overflow, sizeof(int)));
    CK(h, pool_malloc(&h->d_gid, (size_t)h->vcap * sizeof(int)));
    CK(h, pool_malloc(&h->d_nvac, sizeof(int)));
    CK(h, pool_malloc(&h->d_free, (size_t)h->vcap * sizeof(int)));
    CK(h, pool_malloc(&h->d_fcnt, 4 * sizeof(int)));
    CK(h, cudaMemset(h->d_fcnt, 0, 4 * sizeof(int)));
    h->S.freelist = h->d_free;
    h->S.fcnt = h->d_fcnt;
    CK(h, cudaMemset(h->d_nlog, 0, sizeof(unsigned long long)));
    CK(h, cudaMemset(h->d_dist_overflow, 0, sizeof(int)));
    CK(h, cudaMemset(h->d_send, 0, std::max<size_t>(2, np) * per * sizeof(int4)));
    const int nloc = (int)h->nvac;
    CK(h, cudaMemcpy(h->d_nvac, &nloc, sizeof(int), cudaMemcpyHostToDevice));
    h->S.log = h->d_log;
    h->S.nlog = h->d_nlog;
    h->S.gid = h->d_gid;
    // global slot ids: rank of the vacancy's global canonical site index among all ranks' vacancies
    std::vector<int4> v((size_t)std::max<int64_t>(h->nvac, 1));
    if (h->nvac) CK(h, cudaMemcpy(v.data(), h->d_vac, (size_t)h->nvac * sizeof(int4), cudaMemcpyDeviceToHost));
    std::vector<long long> mine((size_t)h->nvac);
    for (int64_t i = 0; i < h->nvac; ++i) {
        const int4 p = v[(size_t)i];
        const long long gx = (p.y >> 1) + h->S.O[0], gy = (p.z >> 1) + h->S.O[1], gz = (p.w >> 1) + h->S.O[2];
        mine[(size_t)i] = 2 * (gx + (long long)h->S.Gc[0] * (gy + (long long)h->S.Gc[1] * gz)) + (p.y & 1);
    }
    long long *d_cnt = nullptr, *d_all = nullptr, *d_mine = nullptr, *d_gath = nullptr;
    CK(h, pool_malloc(&d_cnt, sizeof(long long)));
    CK(h, pool_malloc(&d_all, c.world * sizeof(long long)));
    const long long cnt = h->nvac;
    CK(h, cudaMemcpy(d_cnt, &cnt, sizeof(long long), cudaMemcpyHostToDevice));
    NCK(h, ncclAllGather(d_cnt, d_all, 1, ncclInt64, h->comm, h->stream));
    std::vector<long long> counts(c.world);
    CK(h, cudaMemcpyAsync(counts.data(), d_all, c.world * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    long long mx = 1;
    for (long long x : counts) mx = std::max(mx, x);
    std::vector<long long> pad((size_t)mx, LLONG_MAX);
    std::copy(mine.begin(), mine.end(), pad.begin());
    CK(h, pool_malloc(&d_mine, (size_t)mx * sizeof(long long)));
    CK(h, pool_malloc(&d_gath, (size_t)mx * c.world * sizeof(long long)));
    CK(h, cudaMemcpy(d_mine, pad.data(), (size_t)mx * sizeof(long long), cudaMemcpyHostToDevice));
    NCK(h, ncclAllGather(d_mine, d_gath, (size_t)mx, ncclInt64, h->comm, h->stream));
    std::vector<long long> all((size_t)mx * c.world);
    CK(h, cudaMemcpyAsync(all.data(), d_gath, all.size() * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    cudaFree(d_cnt); cudaFree(d_all); cudaFree(d_mine); cudaFree(d_gath);
    all.erase(std::remove(all.begin(), all.end(), LLONG_MAX), all.end());
    std::sort(all.begin(), all.end());
    std::vector<int> gid((size_t)std::max<int64_t>(h->nvac, 1));
    for (int64_t i = 0; i < h->nvac; ++i)
        gid[(size_t)i] = (int)(std::lower_bound(all.begin(), all.end(), mine[(size_t)i]) - all.begin());
    if (h->nvac) CK(h, cudaMemcpy(h->d_gid, gid.data(), (size_t)h->nvac * sizeof(int), cudaMemcpyHostToDevice));
    const char* ex = std::getenv("AKMC_EXCHANGE");
    if (ex && std::strcmp(ex, "shift") == 0) {
        h->shift = true;
        h->slistcap = h->S.logcap + 6 * (h->DP.cap + 1);
        CK(h, pool_malloc(&h->d_slist, (size_t)h->slistcap * sizeof(int4)));
        CK(h, pool_malloc(&h->d_nslist, sizeof(int)));
    } else if (!(ex && std::strcmp(ex, "nccl") == 0) &&
               2 * std::max(h->DP.G[0], std::max(h->DP.G[1], h->DP.G[2])) < 65536) {
        // (the tagged mailbox entries carry 16-bit global half-cell coordinates; larger global lattices use NCCL)
        const int prc = setup_p2p(h);
        if (prc != AKMC_OK) return prc;
    }
    const auto tv2 = std::chrono::steady_clock::now();
    const int rc = halo_fill(h);
    const auto tv3 = std::chrono::steady_clock::now();
    if (std::getenv("AKMC_VERBOSE"))
        std::fprintf(stderr, "[akmc init_multi rank %d] comm init %.3f s, ids %.3f s, halo fill %.3f s\n", c.rank,
                     std::chrono::duration<double>(tv1 - tv0).count(), std::chrono::duration<double>(tv2 - tv1).count(),
                     std::chrono::duration<double>(tv3 - tv2).count());
    return rc;
}

} // namespace

extern "C" {

const char* akmc_version(void) { return "akmc-b200 0.1 sm_100a"; }

const char* akmc_last_error(const akmc_handle* h) { return h ? h->err.c_str() : g_init_error.c_str(); }

int akmc_init(const akmc_config* cfg, const uint8_t* species, const double* eps, const double* E0, const double* mlp,
              akmc_handle** out)
{
    g_init_error.clear();
    if (!cfg || !species || !out) return fail(nullptr, AKMC_ERR_INVALID, "null argument");
    std::string why;
    int rc = validate(cfg, eps, E0, mlp, why);
    if (rc != AKMC_OK) return fail(nullptr, rc, why);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, AKMC_ERR_CUDA, "no CUDA device available (the AKMC path has no CPU fallback)");
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10 || prop.minor != 0)
        return fail(nullptr, AKMC_ERR_CUDA, "device is not sm_100 (B200); this library is built for sm_100a only");

    akmc_handle* h = new akmc_handle();
    h->cfg = *cfg;
    h->dev = dev;
    h->sub = cfg->domain_cells[0] != 0;
    h->nvox = cfg->n_voxels;
    h->multi = cfg->world > 1;
    h->rc[0] = cfg->rank % cfg->gpu_grid[0];
    h->rc[1] = (cfg->rank / cfg->gpu_grid[0]) % cfg->gpu_grid[1];
    h->rc[2] = cfg->rank / (cfg->gpu_grid[0] * cfg->gpu_grid[1]);
    for (int a = 0; a < 3; ++a) {
        h->F.L[a] = cfg->cells[a];
        h->F.Ls[a] = (cfg->cells[a] + 2 * kHalo + 3) & ~3;               // bricks of 4 cells
        h->F.NB[a] = h->F.Ls[a] / 4;
        h->F.wrap[a] = cfg->gpu_grid[a] == 1 ? 1 : 0;                   // else the halo mirrors a neighbour rank
        h->S.O[a] = h->rc[a] * cfg->cells[a];
        h->S.Gc[a] = cfg->gpu_grid[a] * cfg->cells[a];
        h->DP.O[a] = h->S.O[a];
        h->DP.G[a] = h->S.Gc[a];
        h->S.Lb[a] = cfg->cells[a];
        h->S.dec[a] = cfg->gpu_grid[a] > 1 ? 1 : 0;
    }
    h->F.sites = 128LL * h->F.NB[0] * h->F.NB[1] * h->F.NB[2];          // storage bytes per voxel
    h->csites = 2LL * cfg->cells[0] * cfg->cells[1] * cfg->cells[2];    // canonical sites per voxel
    h->sites = h->csites * cfg->n_voxels;
    h->ssites = h->F.sites * cfg->n_voxels;
    if (!build_geometry(h->G)) { delete h; return fail(nullptr, AKMC_ERR_RUNTIME, "geometry table construction failed"); }
    // physical parameters
    if (eps) {
        for (int s = 0; s < 2; ++s)
            for (int X = 0; X < kSpecies; ++X)
                for (int y = 0; y < kSpecies; ++y) {
                    const double* e = eps + s * kSpecies * kSpecies;
                    const double d = e[X * kSpecies + y] - e[kVac * kSpecies + y];
                    const double dfe = e[X * kSpecies + kFe] - e[kVac * kSpecies + kFe];
                    h->P.Dp[s][X][y] = d - dfe;
                }
    }
    for (int a = 0; a < kSpecies; ++a) h->P.E0[a] = E0 ? E0[a] : 0.0;
    h->have_pair = eps != nullptr && E0 != nullptr;
    h->P.kT = cfg->kB * cfg->temperature_K;
    h->P.inv_kT = 1.0 / h->P.kT;
    h->P.nu0 = cfg->nu0;

#define CKI(x)                                                                                                \
    do {                                                                                                      \
        cudaError_t e_ = (x);                                                                                 \
        if (e_ != cudaSuccess) {                                                                              \
            std::string m_ = std::string(#x) + ": " + cudaGetErrorString(e_);                               \
            free_all(h); delete h;                                                                            \
            return fail(nullptr, AKMC_ERR_CUDA, m_);                                                          \
        }                                                                                                     \
    } while (0)

    h->num_sms = prop.multiProcessorCount;
    // AKMC_VERBOSE: host wall time of the init stages (where bench.py's e2e init time goes)
    const bool verbose = std::getenv("AKMC_VERBOSE") != nullptr;
    auto t_lap = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!verbose) return;
        cudaDeviceSynchronize();
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[akmc init] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t_lap).count());
        t_lap = t;
    };
    CKI(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    lap("context + stream");
    CKI(pool_malloc(&h->d_species, (size_t)h->sites));        // canonical upload buffer (temporary)
    lap("malloc canonical buffer");
    CKI(cudaMemcpy(h->d_species, species, (size_t)h->sites, cudaMemcpyHostToDevice));
    lap("H2D lattice");
    CKI(pool_malloc(&h->d_ctr, sizeof(DevCounters)));
    CKI(cudaMemset(h->d_ctr, 0, sizeof(DevCounters)));
    CKI(cudaMallocHost(&h->h_ctr, sizeof(DevCounters)));

    // a0: vacancy registry by a device scan; slots = vacancies in ascending global site order
    {
        const long long nwords = h->sites / 16;                 // sites is a multiple of 128
        const unsigned nblk = blocks_for(nwords, kScanThreads);
        int* d_bc = nullptr;
        unsigned int* d_max = nullptr;
        long long* d_tot = nullptr;
        CKI(pool_malloc(&d_bc, (size_t)nblk * sizeof(int)));
        h->d_iscratch = d_bc;                                    // freed with the handle on error
        CKI(pool_malloc(&d_max, sizeof(unsigned int) + sizeof(long long) * 2));
        h->d_overflow = reinterpret_cast<unsigned long long*>(d_max);
        d_tot = reinterpret_cast<long long*>(reinterpret_cast<char*>(d_max) + 8);
        CKI(cudaMemset(d_max, 0, sizeof(unsigned int) + sizeof(long long) * 2));
        const uint4* sp4 = reinterpret_cast<const uint4*>(h->d_species);
        scan_count_kernel<<<nblk, kScanThreads, 0, h->stream>>>(sp4, nwords, d_bc, d_max);
        scan_blocks_kernel<<<1, 1024, 0, h->stream>>>(d_bc, (int)nblk, d_tot);
        CKI(cudaGetLastError());
        unsigned int maxcode = 0;
        long long total = 0;
        CKI(cudaMemcpyAsync(&maxcode, d_max, sizeof(unsigned int), cudaMemcpyDeviceToHost, h->stream));
        CKI(cudaMemcpyAsync(&total, d_tot, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
        CKI(cudaStreamSynchronize(h->stream));
        if (maxcode > (unsigned)kVac) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_INVALID, "species code > 6 in the lattice"); }
        h->nvac = total;
        if ((double)h->nvac > 0.01 * (double)h->sites) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_INVALID, "vacancies exceed 1% of sites (S:48)"); }
        if (h->nvac > INT32_MAX / 8) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_INVALID, "too many vacancies"); }
        h->vcap = (int)std::max<int64_t>(h->nvac, 1);
        if (cfg->world > 1) {
            // arrivals from other ranks need spare slots (departed slots are reused, akmc_dist.cuh FreeList);
            // AKMC_VCAP_SPARE (tests) shrinks the spare to exercise the reuse
            int64_t spare = 65536;
            if (const char* sv = std::getenv("AKMC_VCAP_SPARE")) spare = std::max<int64_t>(0, std::atoll(sv));
            const int64_t want = h->nvac + std::max<int64_t>(h->nvac, 0) + spare;
            if (want > INT32_MAX / 16) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_INVALID, "too many vacancies per rank for the slot capacity"); }
            h->vcap = (int)std::max<int64_t>(want, 1);
        }
        CKI(pool_malloc(&h->d_vac, (size_t)h->vcap * sizeof(int4)));
        // slots beyond nvac (vcap >= 1 even with no vacancy; multi-rank spare capacity) start departed (x < 0):
        // the activation reads vcap slots and must never see an uninitialised record as a vacancy
        CKI(cudaMemsetAsync(h->d_vac, 0xFF, (size_t)h->vcap * sizeof(int4), h->stream));
        scan_write_kernel<<<nblk, kScanThreads, 0, h->stream>>>(sp4, nwords, d_bc, h->F, h->d_vac);
        CKI(pool_malloc(&h->d_vstart, (h->nvox + 1) * sizeof(int)));
        vstart_kernel<<<blocks_for(h->nvox + 1, 128), 128, 0, h->stream>>>(h->d_vac, (int)h->nvac, h->nvox, h->d_vstart);
        CKI(cudaGetLastError());
        CKI(cudaStreamSynchronize(h->stream));
        cudaFree(d_bc);
        cudaFree(d_max);
        lap("vacancy scan");
        if (!h->sub) {
            unsigned long long* d_comp = nullptr;
            CKI(pool_malloc(&d_comp, (size_t)h->nvox * 8 * sizeof(unsigned long long)));
            CKI(cudaMemsetAsync(d_comp, 0, (size_t)h->nvox * 8 * sizeof(unsigned long long), h->stream));
            const unsigned bx = (unsigned)std::min<long long>(64, std::max<long long>(1, h->csites / 16 / 256));
            voxel_comp_kernel<<<dim3(bx, (unsigned)h->nvox), 256, 0, h->stream>>>(h->d_species, h->csites, d_comp);
            h->comp.assign((size_t)h->nvox * 8, 0ull);
            CKI(cudaMemcpyAsync(h->comp.data(), d_comp, h->comp.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                h->stream));
            CKI(cudaStreamSynchronize(h->stream));
            cudaFree(d_comp);
        }
        // storage layout with halo ghosts (periodic images)
        uint8_t* st = nullptr;
        CKI(pool_malloc(&st, (size_t)h->ssites));
        lap("malloc storage");
        const long long nlines = 16ll * h->F.NB[0] * h->F.NB[1] * h->F.NB[2] * h->nvox;
        scatter_storage_kernel<<<blocks_for(nlines, 256), 256, 0, h->stream>>>(h->d_species, st, h->F, h->nvox);
        const cudaError_t es = cudaStreamSynchronize(h->stream);
        cudaFree(h->d_species);
        h->d_species = st;
        CKI(es);
        h->d_iscratch = nullptr;
        h->d_overflow = nullptr;
    }
    lap("scatter to bricks");
    const size_t nv = (size_t)h->vcap;
    CKI(pool_malloc(&h->d_rates, nv * 8 * sizeof(double)));
    CKI(pool_malloc(&h->d_E, nv * 8 * sizeof(double)));
    CKI(pool_malloc(&h->d_R, nv * sizeof(double)));
    CKI(pool_malloc(&h->d_scratch, (4 * nv + 64) * sizeof(double)));
    CKI(pool_malloc(&h->d_iscratch, (nv + 16) * sizeof(int)));
    CKI(pool_malloc(&h->d_clock, h->nvox * sizeof(double)));
    CKI(cudaMemset(h->d_clock, 0, h->nvox * sizeof(double)));
    CKI(pool_malloc(&h->d_nev, h->nvox * sizeof(long long)));
    CKI(cudaMemset(h->d_nev, 0, h->nvox * sizeof(long long)));
    CKI(pool_malloc(&h->d_term, h->nvox * sizeof(int)));
    CKI(cudaMemset(h->d_term, 0, h->nvox * sizeof(int)));
    CKI(pool_malloc(&h->d_overflow, sizeof(unsigned long long)));
    CKI(cudaMemset(h->d_overflow, 0, sizeof(unsigned long long)));
    if (h->sub) {
        for (int a = 0; a < 3; ++a) {
            h->S.D[a] = cfg->domain_cells[a];
            h->S.ND[a] = h->S.Gc[a] / cfg->domain_cells[a];             // global domain grid (A16 ids)
        }
        h->S.ndom_vox = (long long)h->S.ND[0] * h->S.ND[1] * h->S.ND[2];
        h->S.window = cfg->window_s;
        h->S.seed = cfg->seed;
        h->ndom_total = h->S.ndom_vox * h->nvox;
        if (h->ndom_total >= 0xFFFFFFFFll) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_INVALID, "too many domains for 32-bit domain ids (A16)"); }
        CKI(pool_malloc(&h->d_dmin, h->ndom_total * sizeof(int)));
        CKI(pool_malloc(&h->d_head, h->ndom_total * sizeof(int)));
        fill_int_kernel<<<blocks_for(h->ndom_total, 256), 256, 0, h->stream>>>(h->d_dmin, h->ndom_total, INT_MAX);
        fill_int_kernel<<<blocks_for(h->ndom_total, 256), 256, 0, h->stream>>>(h->d_head, h->ndom_total, -1);
        CKI(cudaGetLastError());
        CKI(pool_malloc(&h->d_next, nv * sizeof(int)));
        CKI(pool_malloc(&h->d_members, nv * sizeof(int)));
        CKI(pool_malloc(&h->d_mpos, nv * sizeof(int4)));
        CKI(pool_malloc(&h->d_rows, nv * sizeof(int)));
        CKI(pool_malloc(&h->d_segs, nv * sizeof(Segment)));
        CKI(pool_malloc(&h->d_mactive, nv));
        CKI(pool_malloc(&h->d_phase, 8 * sizeof(PhaseInfo)));
        CKI(cudaMallocHost(&h->h_phase, 8 * sizeof(PhaseInfo)));
    }
    lap("per-vacancy / domain buffers");
    if (h->multi) {
        rc = init_multi(h);
        if (rc != AKMC_OK) { std::string m = h->err; free_all(h); delete h; return fail(nullptr, rc, m); }
    }
    if (cfg->barrier_model == AKMC_MODEL_MLP) {
        const size_t n = 448 * kHid + kHid + kHid * kHid + kHid + kHid * 8 + 8;
        CKI(pool_malloc(&h->d_mlp, n * sizeof(double)));
        CKI(cudaMemcpy(h->d_mlp, mlp, n * sizeof(double), cudaMemcpyHostToDevice));
        rc = prepare_engine_weights(h, mlp);
        if (rc != AKMC_OK) { std::string m = h->err; free_all(h); delete h; return fail(nullptr, rc, m); }
    }
    lap("multi-rank setup + weights");
    h->tc = cfg->barrier_model == AKMC_MODEL_MLP && (cfg->precision == AKMC_PREC_FP32 || cfg->precision == AKMC_PREC_FP16_FAST);
    h->engine = std::getenv("AKMC_LEGACY_LOOP") == nullptr;
    if (h->sub) {
        // the phase engine holds at most kRowCap vacancies of one competing set (domain, active sector) in a CTA;
        // a sector with more sites than that could exceed it, so such configurations run the grid-synchronous
        // inner loop (any set size; same selection arithmetic, same evaluator -> same trajectory bits)
        const long long sec_sites = 2LL * (cfg->domain_cells[0] / 2) * (cfg->domain_cells[1] / 2) * (cfg->domain_cells[2] / 2);
        if (sec_sites > kRowCap) h->engine = false;
    }
    if (const char* he = std::getenv("AKMC_HOT_EVENTS")) h->hot_events = std::atof(he);   // A/B knob (0: off)
    if (h->multi && h->p2p && !h->shift && h->engine) {
        // opt-in (measured slower on C5): AKMC_OVERLAP=1
        const char* ov = std::getenv("AKMC_OVERLAP");
        if (ov && std::strcmp(ov, "1") == 0) {
            int lo = 0, hi = 0;
            CKI(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CKI(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi));
            CKI(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
            CKI(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
            CKI(pool_malloc(&h->d_segs2, (size_t)h->vcap * sizeof(Segment)));
            CKI(pool_malloc(&h->d_bdom, (size_t)h->vcap * sizeof(long long)));
            h->overlap_ok = true;
        }
    }
    CKI(engine_setup());
    CKI(bulk_setup());
    CKI(world_setup());
    h->bulk = std::getenv("AKMC_EVAL_ENGINE") == nullptr;
    if (h->tc) {
        h->n_clusters = engine_max_clusters();
        if (h->n_clusters <= 0) { free_all(h); delete h; return fail(nullptr, AKMC_ERR_CUDA, "no co-resident 8-CTA cluster for the evaluator"); }
    }
    CKI(pool_malloc(&h->d_cursor, sizeof(unsigned int)));
    if (std::getenv("AKMC_WATCHDOG")) {
        CKI(cudaHostAlloc(&h->h_watch, 4096 * 8 * sizeof(int), cudaHostAllocMapped));
        std::memset(h->h_watch, 0, 4096 * 8 * sizeof(int));
        CKI(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_watch), h->h_watch, 0));
    }
    {
        const int ncl = std::max(h->n_clusters, 1) + 1;
        CKI(pool_malloc(&h->d_stage, (size_t)ncl * kClusterN * 2 * 65536));
        CKI(pool_malloc(&h->d_wstore, (size_t)std::max(h->num_sms, ncl * kClusterN) * kRowCap * kWin));
    }
    CKI(pool_malloc(&h->d_memo, (size_t)h->vcap * 2 * sizeof(MemoEntry)));
    CKI(cudaMemset(h->d_memo, 0xFF, (size_t)h->vcap * 2 * sizeof(MemoEntry)));   // key 0xFF..: empty
    {
        // per-voxel kT (uniform until akmc_set_voxel_temperatures); the pointer is fixed for the handle's
        // life, so kernel parameters captured in graphs stay valid when the values change
        const std::vector<double> kT((size_t)h->nvox, h->P.kT), ik((size_t)h->nvox, h->P.inv_kT);
        CKI(pool_malloc(&h->d_kT, 2 * kT.size() * sizeof(double)));
        CKI(cudaMemcpy(h->d_kT, kT.data(), kT.size() * sizeof(double), cudaMemcpyHostToDevice));
        CKI(cudaMemcpy(h->d_kT + h->nvox, ik.data(), ik.size() * sizeof(double), cudaMemcpyHostToDevice));
        h->P.kT_vox = h->d_kT;
        h->P.inv_kT_vox = h->d_kT + h->nvox;
    }
    if (!h->sub) {
        // serial / voxel-batch mode through the engine: one segment per voxel, members = its slots in order
        std::vector<int> vs((size_t)h->nvox + 1);
        CKI(cudaMemcpy(vs.data(), h->d_vstart, vs.size() * sizeof(int), cudaMemcpyDeviceToHost));
        std::vector<Segment> sg((size_t)h->nvox);
        int maxm = 0;
        for (int v = 0; v < h->nvox; ++v) {
            sg[(size_t)v] = Segment{(long long)v, vs[(size_t)v], vs[(size_t)v + 1] - vs[(size_t)v], 0.0, 0u, 1};
            maxm = std::max(maxm, sg[(size_t)v].cnt);
        }
        h->serial_engine = h->engine && maxm <= kRowCap;     // a voxel must fit one CTA's member capacity
        std::vector<int> mem((size_t)std::max<int64_t>(h->nvac, 1));
        for (int64_t i = 0; i < h->nvac; ++i) mem[(size_t)i] = (int)i;
        CKI(pool_malloc(&h->d_segs, sg.size() * sizeof(Segment)));
        CKI(pool_malloc(&h->d_members, mem.size() * sizeof(int)));
        CKI(cudaMemcpy(h->d_members, mem.data(), mem.size() * sizeof(int), cudaMemcpyHostToDevice));
        h->vT.assign((size_t)h->nvox, cfg->temperature_K);
        h->vstart_host = vs;
        rc = order_voxels(h);
        if (rc != AKMC_OK) { std::string m = h->err; free_all(h); delete h; return fail(nullptr, rc, m); }
    }
    CKI(cudaStreamSynchronize(h->stream));
    lap("engine setup + memo + segments");
#undef CKI
    *out = h;
    return AKMC_OK;
}

int akmc_set_stream(akmc_handle* h, void* stream)
{
    if (!h) return AKMC_ERR_RUNTIME;
    CK(h, cudaStreamSynchronize(h->stream));
    h->stream = stream ? (cudaStream_t)stream : h->own_stream;
    return AKMC_OK;
}

__global__ void debug_math_kernel(int fn, const double* __restrict__ x, long long n, double* __restrict__ y)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = fn == 0 ? det_exp(x[i]) : det_log(x[i]);
}

int akmc_debug_math(int32_t fn, const double* x, int64_t n, double* y)
{
    if ((fn != 0 && fn != 1) || n < 0 || (n > 0 && (!x || !y))) return AKMC_ERR_INVALID;
    if (n == 0) return AKMC_OK;
    double* d = nullptr;
    if (pool_malloc(&d, (size_t)n * 2 * sizeof(double)) != cudaSuccess) return AKMC_ERR_CUDA;
    cudaError_t e = cudaMemcpy(d, x, (size_t)n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        debug_math_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256>>>(fn, d, (long long)n, d + n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(y, d + n, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? AKMC_OK : AKMC_ERR_CUDA;
}

int akmc_set_voxel_temperatures(akmc_handle* h, const double* T_K, int32_t n)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (!T_K || n != h->nvox) return fail(h, AKMC_ERR_INVALID, "voxel temperatures: need one per voxel");
    std::vector<double> kT((size_t)n);
    for (int v = 0; v < n; ++v) {
        if (!(T_K[v] > 0.0) || !std::isfinite(T_K[v])) return fail(h, AKMC_ERR_INVALID, "temperature must be > 0 (S:154)");
        kT[(size_t)v] = h->cfg.kB * T_K[v];                  // the same IEEE product as the uniform kT
    }
    std::vector<double> ik((size_t)n);
    for (int v = 0; v < n; ++v) ik[(size_t)v] = 1.0 / kT[(size_t)v];
    CK(h, cudaStreamSynchronize(h->stream));
    CK(h, cudaMemcpy(h->d_kT, kT.data(), kT.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(h->d_kT + h->nvox, ik.data(), ik.size() * sizeof(double), cudaMemcpyHostToDevice));
    // memoised rates were formed at the old temperatures (R7: the memo maps window -> rates at fixed T)
    CK(h, cudaMemset(h->d_memo, 0xFF, (size_t)h->vcap * 2 * sizeof(MemoEntry)));
    if (!h->sub) {
        h->vT.assign(T_K, T_K + n);
        return order_voxels(h);                            // Eq. 10 priority at the new temperatures
    }
    return AKMC_OK;
}

int akmc_set_profiling(akmc_handle* h, int32_t profile)
{
    if (!h) return AKMC_ERR_RUNTIME;
    h->profile = profile ? 1 : 0;
    return AKMC_OK;
}

static int step_serial(akmc_handle* h, int64_t n, bool horizon = false, double t_end = 0.0)
{
    if (h->world) {
        // world-model time mode: policy-logit selection (Eqs. 1-2) and the Eq. 7 clock, one CTA per voxel
        for (int64_t done = 0; done < n;) {
            const int chunk = (int)std::min<int64_t>(n - done, 1 << 30);
            WorldParams w{};
            w.species = h->d_species; w.vac = h->d_vac; w.F = h->F; w.G = h->G; w.P = h->P;
            w.mlp = h->d_mlp; w.tnet = h->d_tnet; w.H = h->world_H; w.tau_act = h->world_tau;
            w.nvox = h->nvox; w.vstart = h->d_vstart; w.n_events = chunk;
            w.nev = h->d_nev; w.term = h->d_term; w.clock = h->d_clock; w.seed = h->cfg.seed; w.ctr = h->d_ctr;
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (h->profile) {                          // CUDA events around the launch (mlp_ms)
                if (h->ev_used + 2 > h->ev.size())
                    for (int i = 0; i < 64; ++i) {
                        cudaEvent_t e;
                        CK(h, cudaEventCreate(&e));
                        h->ev.push_back(e);
                    }
                e0 = h->ev[h->ev_used++];
                e1 = h->ev[h->ev_used++];
                CK(h, cudaEventRecord(e0, h->stream));
            }
            CK(h, launch_world(w, h->num_sms, h->stream));
            if (h->profile) CK(h, cudaEventRecord(e1, h->stream));
            h->total.kernel_launches += 1;
            h->total.mlp_launches += 1;
            done += chunk;
        }
        return AKMC_OK;
    }
    if (h->serial_engine) {
        // all n events of every voxel in one persistent launch (a10; per-voxel Philox counters keep the
        // trajectory identical to event-by-event stepping)
        for (int64_t done = 0; done < n;) {
            const int chunk = (int)std::min<int64_t>(n - done, 1 << 30);
            EngineParams p = engine_params(h, kEnginePhase);
            p.serial = 1;
            p.nseg_host = h->nvox;
            p.n_events = chunk;
            p.nev = h->d_nev;
            p.term = h->d_term;
            p.clock = h->d_clock;
            p.horizon = horizon ? 1 : 0;
            p.t_end = t_end;
            p.ph = nullptr;
            CK(h, cudaMemsetAsync(reinterpret_cast<char*>(h->d_ctr) + offsetof(DevCounters, chunk), 0,
                                  sizeof(unsigned long long), h->stream));
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (h->profile) {
                if (h->ev_used + 2 > h->ev.size())
                    for (int i = 0; i < 64; ++i) {
                        cudaEvent_t e;
                        CK(h, cudaEventCreate(&e));
                        h->ev.push_back(e);
                    }
                e0 = h->ev[h->ev_used++];
                e1 = h->ev[h->ev_used++];
                CK(h, cudaEventRecord(e0, h->stream));
            }
            CK(h, launch_engine(p, h->tc, h->n_clusters, h->num_sms, h->stream));
            if (h->profile) CK(h, cudaEventRecord(e1, h->stream));
            h->total.kernel_launches += 2;
            h->total.mlp_launches += 1;
            done += chunk;
        }
        return AKMC_OK;
    }
    const int nv = (int)h->nvac;
    for (int64_t it = 0; it < n; ++it) {
        int rc = eval_rows(h, nullptr, nullptr, nv, nv, nullptr, h->cfg.precision, h->d_rates, h->d_R, h->d_E);
        if (rc != AKMC_OK) return rc;
        select_serial_kernel<<<blocks_for(h->nvox, 128), 128, 0, h->stream>>>(
            h->d_species, h->d_vac, h->F, h->G, h->nvox, h->d_vstart, h->d_rates, h->d_R, h->d_scratch, h->d_clock,
            h->d_nev, h->d_term, h->cfg.seed, h->d_ctr);
        CK(h, cudaGetLastError());
        h->total.kernel_launches += 1;
        h->total.iterations += 1;
    }
    return AKMC_OK;
}

static void phase_table(const akmc_handle* h, int64_t sweep, PhaseInfo ph[8])
{
    int perm[8];
    sector_permutation(h->cfg.seed, sweep, perm);
    for (int q = 0; q < 8; ++q) {
        ph[q].sector = perm[q];
        ph[q].pad = 0;
        ph[q].phase = 8 * sweep + q;
    }
}

struct PhaseTable8 { PhaseInfo p[8]; };

__global__ void set_phase_kernel(PhaseInfo* dst, PhaseTable8 t)
{
    if (threadIdx.x < 8) dst[threadIdx.x] = t.p[threadIdx.x];
}

// the phase's domain lists and segments from the registry as it stands (a1)
static void enqueue_phase_start(akmc_handle* h, const PhaseInfo* ph, cudaStream_t s)
{
    const int nv = h->vcap;
    const int* nd = h->multi ? h->d_nvac : nullptr;
    const unsigned char* memo = h->engine && h->hot_events > 0.0 ? reinterpret_cast<const unsigned char*>(h->d_memo)
                                                                  : nullptr;
    launch_pdl(activate_kernel, blocks_for(nv, 256), 256, s, (const int4*)h->d_vac, nv, nd, h->S, ph, h->d_dmin,
               h->d_head, h->d_next, h->d_ctr, 0, (long long*)nullptr);
    launch_pdl(segments_kernel, blocks_for(nv, 256), 256, s, (const int4*)h->d_vac, nv, nd, h->S, ph, h->d_dmin,
               h->d_head, (const int*)h->d_next, h->d_segs, h->d_members, h->d_mactive, h->d_ctr, h->d_mpos, memo, nv,
               h->hot_events, 0, (Segment*)nullptr);
}

// dataflow sweep (f1): tile base lists, then ONE engine launch that runs all 8 phases of the sweep, every tile
// starting a phase as soon as its 27 neighbour tiles finished the previous one (akmc_engine.cu)
static int enqueue_df_sweep(akmc_handle* h, cudaStream_t s)
{
    EngineParams p = engine_params(h, kEnginePhase);
    p.ph = h->d_phase;
    p.df = 1;
    p.ntiles = h->df_ntiles;
    for (int a = 0; a < 3; ++a) { p.tdom[a] = h->df_tdom[a]; p.NT[a] = h->df_NT[a]; }
    p.done_phase = h->d_done_phase; p.tile_off = h->d_tile_off; p.tile_mem = h->d_tile_mem;
    p.arr_cnt = h->d_arr_cnt; p.arr_slot = h->d_arr_slot;
    p.ring_cap = h->df_ring_cap; p.ring_slot = h->d_ring_slot; p.ring_pos = h->d_ring_pos; p.ring_key = h->d_ring_key;
    p.members = h->d_ring_slot; p.mpos = h->d_ring_pos;          // segment members live in the per-CTA rings
    p.scratch = h->d_df_scratch; p.iscratch = h->d_df_iscratch;  // trees of > 16 members, by ring index
    p.df_err = h->d_df_err;
    CK(h, launch_df_prep(p, h->d_vac, h->vcap, h->d_tile_cnt, h->d_tile_off, h->d_tile_cur, h->d_tile_mem, s));
    CK(h, launch_engine(p, h->tc, h->n_clusters, h->num_sms, s));
    return AKMC_OK;
}

// the whole phase on the device: activate + segments, then the persistent phase engine runs every domain
// of the phase to the end of its window (a2-a8 without any grid-wide synchronisation)
static int enqueue_phase_engine(akmc_handle* h, const PhaseInfo* ph, cudaStream_t s)
{
    enqueue_phase_start(h, ph, s);
    CK(h, cudaGetLastError());
    EngineParams p = engine_params(h, kEnginePhase);
    p.ph = ph;
    CK(h, launch_engine(p, h->tc, h->n_clusters, h->num_sms, s));
    return AKMC_OK;
}

// one inner iteration (a1 rows, a2-a5 eval, a6-a7 select) on stream s; graph adds the a8 condition kernel
static int enqueue_iteration(akmc_handle* h, const PhaseInfo* ph, cudaStream_t s, bool graph,
                             cudaGraphConditionalHandle cond)
{
    const int nv = h->vcap;
    const unsigned gs = std::min<unsigned>(blocks_for(nv, 128), (unsigned)h->num_sms * 4u);
    const unsigned gr = std::min<unsigned>(blocks_for(nv, 256), (unsigned)h->num_sms * 2u);
    rows_kernel<<<gr, 256, 0, s>>>(h->d_segs, h->d_members, h->d_mactive, h->d_rows, h->d_ctr);
    CK(h, cudaGetLastError());
    const int* nrows_dev = reinterpret_cast<const int*>(reinterpret_cast<char*>(h->d_ctr) + offsetof(DevCounters, nrows));
    cudaStream_t keep = h->stream;
    h->stream = s;
    int rc = eval_rows(h, h->d_rows, nrows_dev, 0, nv, nullptr, h->cfg.precision, h->d_rates, h->d_R, h->d_E);
    h->stream = keep;
    if (rc != AKMC_OK) return rc;
    select_sub_kernel<<<gs, 128, 0, s>>>(h->d_species, h->d_vac, h->F, h->G, h->S, ph, h->d_segs, h->d_members,
                                         h->d_mactive, h->d_rates, h->d_R, h->d_scratch, h->d_iscratch, h->d_ctr);
    CK(h, cudaGetLastError());
    if (graph) {
        loop_cond_kernel<<<1, 1, 0, s>>>(h->d_ctr, cond);
        CK(h, cudaGetLastError());
    }
    return AKMC_OK;
}

// CUDA graph of phases [q0, q1): activate + segments, then a conditional WHILE node whose body is one
// inner iteration (rows, eval, select, condition) -- the a8 loop runs on the device with no host
// synchronisation; the phase table (sector permutation) is a device array updated per sweep.
static void enqueue_exchange_p2p(akmc_handle* h, cudaStream_t s);
static int build_graph(akmc_handle* h, int q0, int q1, bool with_window, cudaGraphExec_t* out, int* launches_out)
{
    cudaStream_t cs = nullptr, bs = nullptr;
    CK(h, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(h, cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
    const int ev_profile = h->profile;
    h->profile = 0;                                  // no event nodes inside the graph
    int rc = AKMC_OK;
    int launches = 0;
    cudaGraph_t g = nullptr;
    auto done = [&](int code) {
        h->profile = ev_profile;
        cudaStreamDestroy(cs);
        cudaStreamDestroy(bs);
        return code;
    };
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return done(fail(h, AKMC_ERR_CUDA, "graph capture begin failed"));
    if (h->df) {
        rc = enqueue_df_sweep(h, cs);
        launches += 5;
        q0 = q1;                                     // (all phases are in the one engine launch)
    }
    for (int q = q0; q < q1 && rc == AKMC_OK; ++q) {
        const PhaseInfo* ph = h->d_phase + q;
        if (h->engine) {
            rc = enqueue_phase_engine(h, ph, cs);
            launches += 3;
            if (h->multi && h->p2p && !h->shift && !h->df && with_window) {   // (a multi-rank handle's sweep graph)
                enqueue_exchange_p2p(h, cs);
                launches += 1;
            }
            continue;
        }
        enqueue_phase_start(h, ph, cs);
        launches += 2;
        cudaStreamCaptureStatus st;
        cudaGraph_t cg = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        if (cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg, &deps, &nd) != cudaSuccess) { rc = fail(h, AKMC_ERR_CUDA, "capture info"); break; }
        cudaGraphConditionalHandle hc;
        if (cudaGraphConditionalHandleCreate(&hc, cg, 1, cudaGraphCondAssignDefault) != cudaSuccess) { rc = fail(h, AKMC_ERR_CUDA, "conditional handle"); break; }
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = hc;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t cn;
        if (cudaGraphAddNode(&cn, cg, deps, nd, &np) != cudaSuccess) { rc = fail(h, AKMC_ERR_CUDA, "conditional node"); break; }
        cudaGraph_t body = np.conditional.phGraph_out[0];
        if (cudaStreamUpdateCaptureDependencies(cs, &cn, 1, cudaStreamSetCaptureDependencies) != cudaSuccess) { rc = fail(h, AKMC_ERR_CUDA, "capture deps"); break; }
        if (cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { rc = fail(h, AKMC_ERR_CUDA, "body capture"); break; }
        rc = enqueue_iteration(h, ph, bs, true, hc);
        cudaGraph_t bout = nullptr;
        cudaStreamEndCapture(bs, &bout);
        launches += 4;
    }
    if (with_window) {
        add_window_kernel<<<blocks_for(h->nvox, 128), 128, 0, cs>>>(h->d_clock, h->nvox, h->cfg.window_s);
        launches += 1;
    }
    const cudaError_t ec = cudaStreamEndCapture(cs, &g);
    if (rc != AKMC_OK) { if (g) cudaGraphDestroy(g); return done(rc); }
    if (ec != cudaSuccess) return done(fail(h, AKMC_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec)));
    const cudaError_t ei = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return done(fail(h, AKMC_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)));
    *launches_out = launches;
    return done(AKMC_OK);
}

// multi-rank: after a phase, send logged boundary writes / departures to the peers and apply theirs
// shift-staged exchange of the phase's deltas: stage x, y, z over the decomposed axes, NCCL send /
// recv with the 1-2 neighbours of the axis; receivers forward what the later stages route on (akmc_route.h)
static int exchange_shift(akmc_handle* h)
{
    const akmc_config& c = h->cfg;
    const int cap = h->DP.cap;
    const size_t per = (size_t)(cap + 1);
    ShiftGeom SG{};
    for (int a = 0; a < 3; ++a) { SG.P[a] = h->rc[a]; SG.L[a] = c.cells[a]; SG.grid[a] = c.gpu_grid[a]; }
    shift_collect_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_log, h->d_nlog, h->S.logcap, h->F, h->DP, h->d_species,
                                                            h->d_slist, h->d_nslist, h->d_dist_overflow);
    CK(h, cudaMemsetAsync(h->d_nlog, 0, sizeof(unsigned long long), h->stream));
    int launches = 2;
    int last = -1;
    for (int a = 0; a < 3; ++a) if (c.gpu_grid[a] > 1) last = a;
    for (int a = 0; a < 3; ++a) {
        const int ndir = route::shift_dirs(c.gpu_grid[a]);
        if (!ndir) continue;
        CK(h, cudaMemsetAsync(h->d_send, 0, sizeof(int4), h->stream));
        if (ndir > 1) CK(h, cudaMemsetAsync(h->d_send + per, 0, sizeof(int4), h->stream));
        shift_pack_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_slist, h->d_nslist, a, SG, h->d_send, cap,
                                                             h->d_dist_overflow);
        int e[3] = {0, 0, 0};
        e[a] = 1;
        const int plus = rank_of(c, h->rc[0] + e[0], h->rc[1] + e[1], h->rc[2] + e[2]);
        const int minus = rank_of(c, h->rc[0] - e[0], h->rc[1] - e[1], h->rc[2] - e[2]);
        NCK(h, ncclGroupStart());
        NCK(h, ncclSend(h->d_send, per * sizeof(int4), ncclChar, plus, h->comm, h->stream));        // d = +1
        NCK(h, ncclRecv(h->d_recv, per * sizeof(int4), ncclChar, minus, h->comm, h->stream));       // their d = +1
        if (ndir > 1) {
            NCK(h, ncclSend(h->d_send + per, per * sizeof(int4), ncclChar, minus, h->comm, h->stream));   // d = -1
            NCK(h, ncclRecv(h->d_recv + per, per * sizeof(int4), ncclChar, plus, h->comm, h->stream));
        }
        NCK(h, ncclGroupEnd());
        shift_unpack_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_recv, ndir, cap, h->F, h->DP, h->d_species, h->d_vac,
                                                               h->d_gid, h->d_nvac, h->vcap, FreeList{h->d_free, h->d_fcnt},
                                                               h->d_slist, h->d_nslist, h->slistcap, a != last,
                                                               h->d_dist_overflow);
        launches += 2;
        h->messages += ndir;
        h->exchange_bytes += (int64_t)(2 * ndir * per * sizeof(int4));
    }
    CK(h, cudaGetLastError());
    h->total.kernel_launches += launches;
    h->exchanges += 1;
    return AKMC_OK;
}

// the per-phase peer-mailbox exchange as one launch (graph-capturable: its epoch lives on the device)
static void enqueue_exchange_p2p(akmc_handle* h, cudaStream_t s)
{
    launch_pdl(exchange_p2p_kernel, kP2PBlocks, 256, s, (const int4*)h->d_log, h->d_nlog, h->S.logcap, h->F, h->DP,
               h->PB, (const int4*)h->d_mbox, h->d_species, h->d_vac, h->d_gid, h->d_nvac, h->vcap,
               FreeList{h->d_free, h->d_fcnt}, h->d_dist_overflow);
}

static int exchange_deltas(akmc_handle* h)
{
    if (h->shift) return exchange_shift(h);
    const int np = h->DP.npeer;
    const size_t per = (size_t)(h->DP.cap + 1);
    h->messages += np;
    if (h->p2p) {
        // deltas straight into the peers' mailboxes over NVLink, flag per peer; wait + apply (akmc_dist.cuh)
        if (h->xchg_mark) {                            // (AKMC_PHASE_TIMING: separate launches, to time pack / unpack)
            pack_p2p_kernel<<<kP2PBlocks, 256, 0, h->stream>>>(h->d_log, h->d_nlog, h->S.logcap, h->F, h->DP, h->d_species,
                                                              h->PB, h->d_dist_overflow);
            CK(h, cudaEventRecord(h->xchg_mark[1], h->stream));
            unpack_p2p_kernel<<<kP2PBlocks, 256, 0, h->stream>>>(h->d_mbox, h->d_pepoch, h->F, h->DP, h->d_species,
                                                                h->d_vac, h->d_gid, h->d_nvac, h->vcap,
                                                                FreeList{h->d_free, h->d_fcnt}, h->d_dist_overflow);
            h->total.kernel_launches += 2;
        } else {
            enqueue_exchange_p2p(h, h->stream);
            h->total.kernel_launches += 1;
        }
        CK(h, cudaGetLastError());
        h->exchanges += 1;
        return AKMC_OK;
    }
    pack_deltas_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_log, h->d_nlog, h->S.logcap, h->F, h->DP,
                                                          h->d_species, h->d_send,
                                                          h->d_dist_overflow);
    CK(h, cudaGetLastError());
    NCK(h, ncclGroupStart());
    for (int r = 0; r < np; ++r) {
        NCK(h, ncclSend(h->d_send + r * per, per * sizeof(int4), ncclChar, h->peer_rank[r], h->comm, h->stream));
        NCK(h, ncclRecv(h->d_recv + r * per, per * sizeof(int4), ncclChar, h->peer_rank[r], h->comm, h->stream));
    }
    NCK(h, ncclGroupEnd());
    unpack_deltas_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_recv, np, h->F, h->DP, h->d_species, h->d_vac, h->d_gid,
                                                            h->d_nvac, h->vcap, FreeList{h->d_free, h->d_fcnt},
                                                            h->d_dist_overflow);
    clear_headers_kernel<<<1, 32, 0, h->stream>>>(h->d_send, np, h->DP.cap, h->d_nlog);
    CK(h, cudaGetLastError());
    h->total.kernel_launches += 3;
    h->exchanges += 1;
    h->exchange_bytes += (int64_t)(2 * np * per * sizeof(int4));
    return AKMC_OK;
}

// host-stepped sublattice loop (used when profiling: CUDA events around every barrier-kernel launch)
// AKMC_WATCHDOG: wait for the stream with a deadline; on expiry print every CTA's last progress word and abort
static void watchdog_wait(akmc_handle* h, const char* where)
{
    if (!h->h_watch) return;
    const auto t0 = std::chrono::steady_clock::now();
    while (cudaStreamQuery(h->stream) == cudaErrorNotReady) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) {
            std::fprintf(stderr, "[akmc watchdog] %s: engine did not finish in 20 s; CTA: it code a b nrun drained npend phase\n", where);
            for (int b = 0; b < 4096; ++b) {
                const volatile int* w = h->h_watch + b * 8;
                if (w[1] == 0 && w[0] == 0) continue;
                std::fprintf(stderr, "  cta %4d: %d %d %d %d %d %d %d %d\n", b, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
            }
            std::fflush(stderr);
            std::abort();
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
}

static int step_sublattice_host(akmc_handle* h, int64_t n)
{
    for (int64_t sw = 0; sw < n; ++sw) {
        PhaseTable8 t;
        phase_table(h, h->sweep, t.p);
        set_phase_kernel<<<1, 32, 0, h->stream>>>(h->d_phase, t);
        h->total.kernel_launches += 1;
        for (int q = 0; q < 8; ++q) {
            const PhaseInfo* ph = h->d_phase + q;
            if (h->df) {
                if (q > 0) continue;
                if (h->ev_used + 2 > h->ev.size())
                    for (int i = 0; i < 64; ++i) {
                        cudaEvent_t e;
                        CK(h, cudaEventCreate(&e));
                        h->ev.push_back(e);
                    }
                cudaEvent_t e0 = h->ev[h->ev_used++], e1 = h->ev[h->ev_used++];
                CK(h, cudaEventRecord(e0, h->stream));
                const int rc = enqueue_df_sweep(h, h->stream);
                if (rc != AKMC_OK) return rc;
                watchdog_wait(h, "dataflow sweep");
                CK(h, cudaEventRecord(e1, h->stream));
                h->total.kernel_launches += 5;
                h->total.mlp_launches += 1;
                continue;
            }
            if (h->engine) {
                cudaEvent_t e0 = nullptr, e1 = nullptr;
                if (h->ev_used + 2 > h->ev.size()) {
                    for (int i = 0; i < 64; ++i) {
                        cudaEvent_t e;
                        CK(h, cudaEventCreate(&e));
                        h->ev.push_back(e);
                    }
                }
                e0 = h->ev[h->ev_used++];
                e1 = h->ev[h->ev_used++];
                CK(h, cudaEventRecord(e0, h->stream));
                const int rc = enqueue_phase_engine(h, ph, h->stream);
                if (rc != AKMC_OK) return rc;
                watchdog_wait(h, "phase");
                CK(h, cudaEventRecord(e1, h->stream));
                h->total.kernel_launches += 3;
                h->total.mlp_launches += 1;
                if (h->multi) {
                    const bool xt = h->d_phase_cycles && h->p2p && !h->shift;   // AKMC_PHASE_TIMING: split the exchange
                    if (xt) {
                        if (h->xev_used + 3 > h->xev.size())
                            for (int i = 0; i < 48; ++i) {
                                cudaEvent_t e;
                                CK(h, cudaEventCreate(&e));
                                h->xev.push_back(e);
                            }
                        h->xchg_mark = h->xev.data() + h->xev_used;
                        h->xev_used += 3;
                        CK(h, cudaEventRecord(h->xchg_mark[0], h->stream));
                    }
                    const int rc2 = exchange_deltas(h);
                    if (rc2 != AKMC_OK) return rc2;
                    if (xt) { CK(h, cudaEventRecord(h->xchg_mark[2], h->stream)); h->xchg_mark = nullptr; }
                }
                continue;
            }
            enqueue_phase_start(h, ph, h->stream);
            CK(h, cudaGetLastError());
            h->total.kernel_launches += 2;
            for (;;) {
                int rc = enqueue_iteration(h, ph, h->stream, false, 0);
                if (rc != AKMC_OK) return rc;
                h->total.kernel_launches += 2;
                h->total.iterations += 1;
                CK(h, cudaMemcpyAsync(h->h_ctr, h->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, h->stream));
                CK(h, cudaStreamSynchronize(h->stream));
                const bool more = h->h_ctr->nrun > 0;
                CK(h, cudaMemsetAsync(reinterpret_cast<char*>(h->d_ctr) + offsetof(DevCounters, nrun), 0,
                                      sizeof(unsigned long long), h->stream));
                CK(h, cudaMemsetAsync(reinterpret_cast<char*>(h->d_ctr) + offsetof(DevCounters, nrows), 0,
                                      sizeof(unsigned long long), h->stream));
                if (!more) break;
            }
            if (h->multi) {
                const int rc = exchange_deltas(h);
                if (rc != AKMC_OK) return rc;
            }
        }
        add_window_kernel<<<blocks_for(h->nvox, 128), 128, 0, h->stream>>>(h->d_clock, h->nvox, h->cfg.window_s);
        CK(h, cudaGetLastError());
        h->total.kernel_launches += 1;
        h->sweep += 1;
        h->total.sweeps += 1;
    }
    return AKMC_OK;
}

// Multi-rank sweep with the per-phase exchange overlapped.  After phase q the deltas
// are packed into the peers' mailboxes and every domain list of phase q + 1 is built from the registry as it
// stands (stream A); then the receive side -- wait for the peers' deltas of q, apply them, put the arriving
// vacancies into the lists, cut the boundary domains' segments (the first and last domain layer along each
// decomposed axis: the only domains that read the halo or receive arrivals) -- runs on a second stream while
// phase q + 1's engine already runs the interior domains on stream A; the engine takes the boundary segments once
// they are published (ctr->bready, release / acquire).  Domains of a phase are independent (R6): the trajectory is
// the unoverlapped one bit for bit.
static void enqueue_unpack_p2p(akmc_handle* h, cudaStream_t s, const PhaseInfo* ph_next)
{
    ArrivalActivation act{};
    if (ph_next) {
        act.ph = ph_next; act.S = h->S; act.dmin = h->d_dmin; act.head = h->d_head; act.next = h->d_next;
        act.bdom = h->d_bdom; act.ctr = h->d_ctr;
    }
    unpack_p2p_kernel<<<kP2PBlocks, 256, 0, s>>>(h->d_mbox, h->d_pepoch, h->F, h->DP, h->d_species, h->d_vac,
                                                 h->d_gid, h->d_nvac, h->vcap, FreeList{h->d_free, h->d_fcnt},
                                                 h->d_dist_overflow, act);
    h->xpending = false;
    h->total.kernel_launches += 1;
}

static int step_sublattice_overlap(akmc_handle* h, int64_t n)
{
    const int nv = h->vcap;
    const int np = h->DP.npeer;
    cudaStream_t A = h->stream, B = h->side;
    for (int64_t sw = 0; sw < n; ++sw) {
        PhaseTable8 t;
        phase_table(h, h->sweep, t.p);
        set_phase_kernel<<<1, 32, 0, A>>>(h->d_phase, t);
        for (int q = 0; q < 8; ++q) {
            const PhaseInfo* ph = h->d_phase + q;
            // every domain's member list from the current registry (also resets the phase counters)
            activate_kernel<<<blocks_for(nv, 256), 256, 0, A>>>(h->d_vac, nv, h->d_nvac, h->S, ph, h->d_dmin, h->d_head,
                                                                h->d_next, h->d_ctr, 0, h->d_bdom);
            CK(h, cudaEventRecord(h->ev_fork, A));
            // receive side of the previous exchange + the boundary segments (few blocks: the engine keeps its SMs)
            CK(h, cudaStreamWaitEvent(B, h->ev_fork, 0));
            if (h->xpending) enqueue_unpack_p2p(h, B, ph);
            segments_boundary_kernel<<<4, 256, 0, B>>>(h->d_bdom, h->S, h->d_vac, h->d_dmin, h->d_head,
                                                                    h->d_next, h->d_segs2, h->d_members, h->d_mactive,
                                                                    h->d_ctr, h->d_mpos);
            publish_boundary_kernel<<<1, 32, 0, B>>>(h->d_ctr, ph);
            CK(h, cudaEventRecord(h->ev_join, B));
            // interior segments + the engine on stream A
            segments_kernel<<<blocks_for(nv, 256), 256, 0, A>>>(h->d_vac, nv, h->d_nvac, h->S, ph, h->d_dmin, h->d_head,
                                                                h->d_next, h->d_segs, h->d_members, h->d_mactive, h->d_ctr,
                                                                h->d_mpos,
                                                                h->hot_events > 0.0
                                                                    ? reinterpret_cast<const unsigned char*>(h->d_memo) : nullptr,
                                                                nv, h->hot_events, 1, nullptr);
            EngineParams p = engine_params(h, kEnginePhase);
            p.ph = ph;
            p.overlap = 1;
            p.segs2 = h->d_segs2;
            // (the engine leaves >= 16 SMs to the side stream, whose kernels it may be waiting for)
            const int spare = h->num_sms - 16;
            CK(h, launch_engine(p, h->tc, std::max(1, std::min(h->n_clusters, spare / 4)), spare, A));
            CK(h, cudaStreamWaitEvent(A, h->ev_join, 0));
            // send side of this phase's exchange
            pack_p2p_kernel<<<kP2PBlocks, 256, 0, A>>>(h->d_log, h->d_nlog, h->S.logcap, h->F, h->DP, h->d_species, h->PB,
                                                       h->d_dist_overflow);
            CK(h, cudaGetLastError());
            h->xpending = true;
            h->messages += np;
            h->exchanges += 1;
            h->total.kernel_launches += 6;
            h->total.mlp_launches += 1;
        }
        add_window_kernel<<<blocks_for(h->nvox, 128), 128, 0, A>>>(h->d_clock, h->nvox, h->cfg.window_s);
        CK(h, cudaGetLastError());
        h->total.kernel_launches += 2;
        h->sweep += 1;
        h->total.sweeps += 1;
    }
    if (h->xpending) enqueue_unpack_p2p(h, A, nullptr);   // leave the halo and the registry complete at the call's end
    CK(h, cudaGetLastError());
    return AKMC_OK;
}

static int step_sublattice(akmc_handle* h, int64_t n)
{
    if (h->profile) return step_sublattice_host(h, n);
    if (h->multi && h->overlap_ok && !h->df) return step_sublattice_overlap(h, n);
    int launches_phase = 0;
    // one graph per sweep: a single rank, or ranks exchanging through the peer mailboxes (the exchange kernel's
    // epoch lives on the device, so it replays inside the graph); NCCL / shift exchanges run between phase graphs
    const bool one_graph = !h->multi || (h->p2p && !h->shift && h->engine && !h->df);
    if (one_graph && !h->sweep_exec) {
        const int rc = build_graph(h, 0, 8, true, &h->sweep_exec, &h->graph_launches_per_sweep);
        if (rc != AKMC_OK) return rc;
    }
    if (!one_graph && !h->phase_exec[0]) {
        for (int q = 0; q < 8; ++q) {
            const int rc = build_graph(h, q, q + 1, false, &h->phase_exec[q], &launches_phase);
            if (rc != AKMC_OK) return rc;
        }
        h->graph_launches_per_sweep = 8 * launches_phase;
    }
    for (int64_t sw = 0; sw < n; ++sw) {
        PhaseTable8 t;
        phase_table(h, h->sweep, t.p);
        set_phase_kernel<<<1, 32, 0, h->stream>>>(h->d_phase, t);
        CK(h, cudaGetLastError());
        if (one_graph) {
            CK(h, cudaGraphLaunch(h->sweep_exec, h->stream));
            watchdog_wait(h, "sweep");
            if (h->multi) { h->messages += 8 * h->DP.npeer; h->exchanges += 8; }
        } else {
            for (int q = 0; q < 8; ++q) {
                CK(h, cudaGraphLaunch(h->phase_exec[q], h->stream));
                watchdog_wait(h, "phase graph");
                const int rc = exchange_deltas(h);
                if (rc != AKMC_OK) return rc;
                watchdog_wait(h, "exchange");
            }
            add_window_kernel<<<blocks_for(h->nvox, 128), 128, 0, h->stream>>>(h->d_clock, h->nvox, h->cfg.window_s);
            CK(h, cudaGetLastError());
            h->total.kernel_launches += 1;
        }
        h->total.kernel_launches += 1 + h->graph_launches_per_sweep;   // body kernels counted once per phase
        h->sweep += 1;
        h->total.sweeps += 1;
    }
    return AKMC_OK;
}

// The evaluator's fp16 range guard and the engine's capacity guards count into d_overflow ("must stay 0").  A
// non-zero count means some rate of this call was formed from a clamped activation or some competing set was
// not run: the call fails loudly instead of returning a wrong trajectory with AKMC_OK.
static int check_overflow(akmc_handle* h, const char* where)
{
    unsigned long long ovf = 0;
    CK(h, cudaMemcpyAsync(&ovf, h->d_overflow, sizeof(ovf), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (!ovf) return AKMC_OK;
    CK(h, cudaMemsetAsync(h->d_overflow, 0, sizeof(ovf), h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return fail(h, AKMC_ERR_RUNTIME, std::string(where) + ": " + std::to_string(ovf) +
                " evaluator range / engine capacity overflow(s) (fp16 activation clamp or a competing set beyond the "
                "engine's capacity); the results of this call are invalid");
}

static int step_common(akmc_handle* h, int64_t n, akmc_counters* ctr, bool horizon, double t_end)
{
    const akmc_counters before = h->total;
    CK(h, cudaMemcpyAsync(h->h_ctr, h->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    const DevCounters c0 = *h->h_ctr;
    const auto t0 = std::chrono::steady_clock::now();
    int rc = h->sub ? step_sublattice(h, n) : step_serial(h, n, horizon, t_end);
    if (rc != AKMC_OK) return rc;
    CK(h, cudaMemcpyAsync(h->h_ctr, h->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    rc = harvest_events(h);
    if (rc != AKMC_OK) return rc;
    const DevCounters c1 = *h->h_ctr;
    const auto t1 = std::chrono::steady_clock::now();
    h->total.events += (int64_t)(c1.events - c0.events);
    h->total.hop_evals += (int64_t)(c1.hop_evals - c0.hop_evals);
    h->total.mlp_rows += ((h->engine && h->sub) || h->serial_engine || h->world) ? (int64_t)(c1.mrows - c0.mrows)
                                                                      : (int64_t)(c1.hop_evals - c0.hop_evals) / 8;
    h->total.clamps += (int64_t)(c1.clamps - c0.clamps);
    h->total.terminal_voxels += (int64_t)(c1.terminal - c0.terminal);
    h->total.wall_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (ctr) {
        akmc_counters d{};
        d.events = h->total.events - before.events;
        d.hop_evals = h->total.hop_evals - before.hop_evals;
        d.iterations = h->total.iterations - before.iterations;
        d.clamps = h->total.clamps - before.clamps;
        d.terminal_voxels = h->total.terminal_voxels - before.terminal_voxels;
        d.sweeps = h->total.sweeps - before.sweeps;
        d.kernel_launches = h->total.kernel_launches - before.kernel_launches;
        d.mlp_launches = h->total.mlp_launches - before.mlp_launches;
        d.mlp_rows = h->total.mlp_rows - before.mlp_rows;
        d.mlp_ms = h->total.mlp_ms - before.mlp_ms;
        d.wall_ms = h->total.wall_ms - before.wall_ms;
        *ctr = d;
    }
    rc = check_overflow(h, "akmc_step");
    if (rc != AKMC_OK) return rc;
    if (h->df) {
        int e = 0;
        CK(h, cudaMemcpy(&e, h->d_df_err, sizeof(int), cudaMemcpyDeviceToHost));
        if (e) {
            CK(h, cudaMemset(h->d_df_err, 0, sizeof(int)));
            return fail(h, AKMC_ERR_RUNTIME, "dataflow sweep: tile arrival / activation ring capacity exceeded (" +
                                                 std::to_string(e) + "); the results of this call are invalid");
        }
    }
    if (h->multi) {
        int ovf = 0;
        CK(h, cudaMemcpy(&ovf, h->d_dist_overflow, sizeof(int), cudaMemcpyDeviceToHost));
        if (ovf & kExchangeTimeout) return fail(h, AKMC_ERR_RUNTIME, "halo exchange timeout: a peer rank did not publish its deltas within 30 s");
        if (ovf) return fail(h, AKMC_ERR_RUNTIME, "halo exchange buffer overflow (" + std::to_string(ovf) + " entries)");
    }
    if (c1.terminal != c0.terminal) return fail(h, AKMC_TERMINAL, "a competing set has no feasible event (S:199)");
    return AKMC_OK;
}

int akmc_step(akmc_handle* h, int64_t n, akmc_counters* ctr)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (n < 0) return fail(h, AKMC_ERR_INVALID, "n must be >= 0");
    return step_common(h, n, ctr, false, 0.0);
}

int akmc_run_until(akmc_handle* h, double t_end_s, int64_t max_events, akmc_counters* ctr)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (h->sub) return fail(h, AKMC_ERR_INVALID, "akmc_run_until: serial (voxel) mode only");
    if (h->world) return fail(h, AKMC_ERR_INVALID, "akmc_run_until: not available in world-model mode");
    if (!h->serial_engine) return fail(h, AKMC_ERR_INVALID, "akmc_run_until: needs the engine path (AKMC_LEGACY_LOOP unset, "
                                                            "a voxel's vacancies fit one engine CTA)");
    if (!std::isfinite(t_end_s) || max_events < 0 || max_events > (1LL << 30))
        return fail(h, AKMC_ERR_INVALID, "akmc_run_until: bad t_end or max_events (0 .. 2^30)");
    return step_common(h, max_events, ctr, true, t_end_s);
}

struct VacRec { int64_t gid, site; int slot; };

// live vacancies of this handle: (global slot id, global canonical site, local slot), sorted by gid
static int collect_vacancies(akmc_handle* h, std::vector<VacRec>& out)
{
    out.clear();
    int n = (int)h->nvac;
    if (h->multi) CK(h, cudaMemcpy(&n, h->d_nvac, sizeof(int), cudaMemcpyDeviceToHost));
    n = std::min(n, h->vcap);
    if (n <= 0) return AKMC_OK;
    std::vector<int4> v((size_t)n);
    std::vector<int> g((size_t)n);
    CK(h, cudaMemcpy(v.data(), h->d_vac, (size_t)n * sizeof(int4), cudaMemcpyDeviceToHost));
    if (h->multi) CK(h, cudaMemcpy(g.data(), h->d_gid, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
        const int4 p = v[(size_t)i];
        if (p.x < 0) continue;
        const int64_t gx = (p.y >> 1) + h->S.O[0], gy = (p.z >> 1) + h->S.O[1], gz = (p.w >> 1) + h->S.O[2];
        const int64_t Gx = h->multi ? h->S.Gc[0] : h->F.L[0], Gy = h->multi ? h->S.Gc[1] : h->F.L[1];
        const int64_t site = (int64_t)p.x * h->csites + 2 * (gx + Gx * (gy + Gy * gz)) + (p.y & 1);
        out.push_back({h->multi ? (int64_t)g[(size_t)i] : (int64_t)i, site, i});
    }
    std::sort(out.begin(), out.end(), [](const VacRec& a, const VacRec& b) { return a.gid < b.gid; });
    return AKMC_OK;
}

int akmc_state(akmc_handle* h, uint8_t* species_out, int64_t* vac_sites_out, int64_t* n_vac_inout, double* clock_s_out,
               akmc_counters* ctr_out)
{
    if (!h) return AKMC_ERR_RUNTIME;
    CK(h, cudaStreamSynchronize(h->stream));
    std::vector<VacRec> vr;
    if (vac_sites_out || n_vac_inout) {
        const int rc = collect_vacancies(h, vr);
        if (rc != AKMC_OK) return rc;
    }
    if (vac_sites_out && (!n_vac_inout || *n_vac_inout < (int64_t)vr.size()))
        return fail(h, AKMC_ERR_INVALID, "vacancy buffer too short");
    if (species_out) {
        if (!h->d_canon) CK(h, pool_malloc(&h->d_canon, (size_t)h->sites));   // kept for later readbacks
        uint8_t* canon = h->d_canon;
        const long long nchunks = (long long)((h->F.L[0] + 3) / 4) * h->F.L[1] * h->F.L[2] * h->nvox;
        gather_canonical_kernel<<<blocks_for(nchunks, 256), 256, 0, h->stream>>>(h->d_species, canon, h->F, h->nvox);
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess) e = cudaMemcpy(species_out, canon, (size_t)h->sites, cudaMemcpyDeviceToHost);
        CK(h, e);
    }
    if (vac_sites_out)
        for (size_t i = 0; i < vr.size(); ++i) vac_sites_out[i] = vr[i].site;
    if (n_vac_inout) *n_vac_inout = (int64_t)vr.size();
    if (clock_s_out) CK(h, cudaMemcpy(clock_s_out, h->d_clock, h->nvox * sizeof(double), cudaMemcpyDeviceToHost));
    if (ctr_out) *ctr_out = h->total;
    return AKMC_OK;
}

int akmc_vacancies(akmc_handle* h, int64_t* gid_out, int64_t* site_out, int64_t* n_inout)
{
    if (!h || !n_inout) return AKMC_ERR_RUNTIME;
    CK(h, cudaStreamSynchronize(h->stream));
    std::vector<VacRec> vr;
    int rc = collect_vacancies(h, vr);
    if (rc != AKMC_OK) return rc;
    if ((gid_out || site_out) && *n_inout < (int64_t)vr.size()) return fail(h, AKMC_ERR_INVALID, "vacancy buffer too short");
    for (size_t i = 0; i < vr.size(); ++i) {
        if (gid_out) gid_out[i] = vr[i].gid;
        if (site_out) site_out[i] = vr[i].site;
    }
    *n_inout = (int64_t)vr.size();
    return AKMC_OK;
}

int akmc_set_world_model(akmc_handle* h, const double* tnet, int32_t hidden, double tau_act)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (h->sub) return fail(h, AKMC_ERR_INVALID, "world-model mode: serial / voxel-batch mode only (domain_cells = 0)");
    if (h->cfg.barrier_model != AKMC_MODEL_MLP || h->cfg.precision != AKMC_PREC_FP64)
        return fail(h, AKMC_ERR_INVALID, "world-model mode: needs the MLP (policy logits) at FP64 precision");
    if (!h->have_pair) return fail(h, AKMC_ERR_INVALID, "world-model mode: eps and E0 must be given at init (physical rates of Eq. 7)");
    if (!tnet || hidden < 1 || hidden > kWorldMaxHidden) return fail(h, AKMC_ERR_INVALID, "world-model mode: bad Poisson-net shape");
    if (!(tau_act > 0.0) || !std::isfinite(tau_act)) return fail(h, AKMC_ERR_INVALID, "world-model mode: tau_act must be > 0 (Eq. 1)");
    const size_t n = (size_t)448 * hidden + 2 * (size_t)hidden + 1;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(tnet[i])) return fail(h, AKMC_ERR_INVALID, "world-model mode: non-finite Poisson-net weight");
    std::vector<int> vs((size_t)h->nvox + 1);
    CK(h, cudaMemcpy(vs.data(), h->d_vstart, vs.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int v = 0; v < h->nvox; ++v)
        if (vs[(size_t)v + 1] - vs[(size_t)v] > kWorldMaxVac)
            return fail(h, AKMC_ERR_INVALID, "world-model mode: more than 64 vacancies in a voxel");
    CK(h, cudaStreamSynchronize(h->stream));
    if (h->d_tnet) { cudaFree(h->d_tnet); h->d_tnet = nullptr; }
    CK(h, pool_malloc(&h->d_tnet, n * sizeof(double)));
    CK(h, cudaMemcpy(h->d_tnet, tnet, n * sizeof(double), cudaMemcpyHostToDevice));
    h->world_H = hidden;
    h->world_tau = tau_act;
    h->world = true;
    return AKMC_OK;
}

int akmc_set_dataflow(akmc_handle* h, int32_t on)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (on && (!h->sub || h->multi || !h->engine))
        return fail(h, AKMC_ERR_INVALID, "dataflow sweeps: single-rank sublattice handles on the phase engine only");
    CK(h, cudaStreamSynchronize(h->stream));
    if (h->sweep_exec) { cudaGraphExecDestroy(h->sweep_exec); h->sweep_exec = nullptr; }
    if (!on) { h->df = false; return AKMC_OK; }
    if (!h->d_done_phase) {
        // tiles of tdom^3 domains: grow the tile edge until every CTA of the persistent grid holds <= kMyTiles tiles
        const int grid = h->tc ? kClusterN * h->n_clusters : h->num_sms;
        int td[3] = {1, 1, 1}, NT[3];
        long long nt = 0;
        for (;;) {
            for (int a = 0; a < 3; ++a) NT[a] = (h->S.ND[a] + td[a] - 1) / td[a];
            nt = (long long)NT[0] * NT[1] * NT[2] * h->nvox;
            if (nt <= (long long)kMyTiles * grid) break;
            int a = 0;
            for (int b = 1; b < 3; ++b) if (NT[b] > NT[a]) a = b;
            if (td[a] >= h->S.ND[a]) return fail(h, AKMC_ERR_INVALID, "dataflow sweeps: too many voxels for the tile capacity");
            td[a] *= 2;
        }
        for (int a = 0; a < 3; ++a) { h->df_tdom[a] = td[a]; h->df_NT[a] = NT[a]; }
        h->df_ntiles = (int)nt;
        h->df_grid = grid;
        const size_t ring = (size_t)grid * h->df_ring_cap;
        CK(h, pool_malloc(&h->d_done_phase, nt * sizeof(long long)));
        CK(h, pool_malloc(&h->d_tile_off, (nt + 1) * sizeof(int)));
        CK(h, pool_malloc(&h->d_tile_cnt, nt * sizeof(int)));
        CK(h, pool_malloc(&h->d_tile_cur, nt * sizeof(int)));
        CK(h, pool_malloc(&h->d_tile_mem, (size_t)h->vcap * sizeof(int)));
        CK(h, pool_malloc(&h->d_arr_cnt, nt * sizeof(int)));
        CK(h, pool_malloc(&h->d_arr_slot, nt * kArrCap * sizeof(int)));
        CK(h, cudaMemset(h->d_arr_slot, 0xFF, nt * kArrCap * sizeof(int)));
        CK(h, pool_malloc(&h->d_ring_slot, ring * sizeof(int)));
        CK(h, pool_malloc(&h->d_ring_pos, ring * sizeof(int4)));
        CK(h, pool_malloc(&h->d_ring_key, ring * sizeof(unsigned long long)));
        CK(h, pool_malloc(&h->d_df_scratch, (4 * ring + 64) * sizeof(double)));
        CK(h, pool_malloc(&h->d_df_iscratch, (ring + 16) * sizeof(int)));
        CK(h, pool_malloc(&h->d_df_err, sizeof(int)));
        CK(h, cudaMemset(h->d_df_err, 0, sizeof(int)));
    }
    h->df = true;
    return AKMC_OK;
}

int akmc_exchange_stats(akmc_handle* h, int64_t* out3)
{
    if (!h || !out3) return AKMC_ERR_INVALID;
    out3[0] = h->exchanges;
    out3[1] = h->messages;
    out3[2] = h->exchange_bytes;
    return AKMC_OK;
}

int akmc_voxel_order(akmc_handle* h, int32_t* order_out)
{
    if (!h || !order_out) return AKMC_ERR_INVALID;
    if (h->sub) return fail(h, AKMC_ERR_INVALID, "akmc_voxel_order: serial (voxel) mode only");
    std::copy(h->vorder.begin(), h->vorder.end(), order_out);
    return AKMC_OK;
}

int akmc_progress(akmc_handle* h, int64_t* nev_out, int64_t* sweep_out)
{
    if (!h) return AKMC_ERR_RUNTIME;
    CK(h, cudaStreamSynchronize(h->stream));
    if (nev_out) {
        static_assert(sizeof(long long) == sizeof(int64_t), "event counter width");
        CK(h, cudaMemcpy(nev_out, h->d_nev, (size_t)h->nvox * sizeof(long long), cudaMemcpyDeviceToHost));
    }
    if (sweep_out) *sweep_out = h->sweep;
    return AKMC_OK;
}

int akmc_restore(akmc_handle* h, const int64_t* vac_sites, int64_t n_vac, const double* clock_s, const int64_t* nev,
                 int64_t sweep)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (h->multi) return fail(h, AKMC_ERR_INVALID, "akmc_restore: single-rank handles only");
    if (sweep < 0) return fail(h, AKMC_ERR_INVALID, "akmc_restore: sweep must be >= 0");
    CK(h, cudaStreamSynchronize(h->stream));
    if (vac_sites) {
        if (n_vac != h->nvac) return fail(h, AKMC_ERR_INVALID, "akmc_restore: vacancy count differs from the lattice's");
        std::vector<VacRec> cur;
        const int rc = collect_vacancies(h, cur);
        if (rc != AKMC_OK) return rc;
        std::vector<int64_t> a((size_t)n_vac), b;
        b.reserve(cur.size());
        for (const VacRec& r : cur) b.push_back(r.site);
        std::copy(vac_sites, vac_sites + n_vac, a.begin());
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        if (a != b || std::adjacent_find(a.begin(), a.end()) != a.end())
            return fail(h, AKMC_ERR_INVALID, "akmc_restore: vac_sites is not the lattice's vacancy set");
        std::vector<int4> v((size_t)std::max<int64_t>(n_vac, 1));
        const int Lx = h->F.L[0], Ly = h->F.L[1];
        for (int64_t i = 0; i < n_vac; ++i) {
            const int64_t site = vac_sites[i];
            const int vox = (int)(site / h->csites);
            const int64_t r = site % h->csites;
            const int bb = (int)(r & 1);
            const int64_t c = r >> 1;
            const int x = (int)(c % Lx), y = (int)((c / Lx) % Ly), z = (int)(c / ((int64_t)Lx * Ly));
            if (i > 0 && vox < v[(size_t)i - 1].x)
                return fail(h, AKMC_ERR_INVALID, "akmc_restore: slots must be grouped by voxel in ascending order");
            v[(size_t)i] = make_int4(vox, 2 * x + bb, 2 * y + bb, 2 * z + bb);
        }
        if (n_vac) CK(h, cudaMemcpy(h->d_vac, v.data(), (size_t)n_vac * sizeof(int4), cudaMemcpyHostToDevice));
    }
    if (clock_s) {
        for (int i = 0; i < h->nvox; ++i)
            if (!std::isfinite(clock_s[i]) || clock_s[i] < 0.0) return fail(h, AKMC_ERR_INVALID, "akmc_restore: bad clock");
        CK(h, cudaMemcpy(h->d_clock, clock_s, (size_t)h->nvox * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (nev) {
        for (int i = 0; i < h->nvox; ++i)
            if (nev[i] < 0) return fail(h, AKMC_ERR_INVALID, "akmc_restore: event counters must be >= 0");
        CK(h, cudaMemcpy(h->d_nev, nev, (size_t)h->nvox * sizeof(long long), cudaMemcpyHostToDevice));
    }
    h->sweep = sweep;
    CK(h, cudaMemset(h->d_term, 0, (size_t)h->nvox * sizeof(int)));
    CK(h, cudaMemset(h->d_memo, 0xFF, (size_t)h->vcap * 2 * sizeof(MemoEntry)));
    return AKMC_OK;
}

int akmc_debug_extended(akmc_handle* h, uint8_t* out)
{
    if (!h || !out) return AKMC_ERR_INVALID;
    CK(h, cudaStreamSynchronize(h->stream));
    SlabRange R{};
    for (int a = 0; a < 3; ++a) { R.lo[a] = -kHalo; R.hi[a] = h->F.L[a] + kHalo; }
    const size_t bytes = 2ull * (h->F.L[0] + 2 * kHalo) * (h->F.L[1] + 2 * kHalo) * (h->F.L[2] + 2 * kHalo);
    uint8_t* d = nullptr;
    CK(h, pool_malloc(&d, bytes));
    pack_slab_kernel<<<h->num_sms * 4, 256, 0, h->stream>>>(h->d_species, h->F, R, d);
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    CK(h, e);
    return AKMC_OK;
}

int akmc_nccl_unique_id(uint8_t* out128)
{
    if (!out128) return AKMC_ERR_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return AKMC_ERR_NCCL;
    std::memset(out128, 0, 128);
    std::memcpy(out128, &id, sizeof(id));
    return AKMC_OK;
}

int akmc_rates(akmc_handle* h, double* rates_out, double* barriers_out)
{
    if (!h) return AKMC_ERR_RUNTIME;
    std::vector<VacRec> vr;
    int rc = collect_vacancies(h, vr);
    if (rc != AKMC_OK) return rc;
    int nslots = (int)h->nvac;
    if (h->multi) CK(h, cudaMemcpy(&nslots, h->d_nvac, sizeof(int), cudaMemcpyDeviceToHost));
    nslots = std::min(nslots, h->vcap);
    if (nslots <= 0 || vr.empty()) return AKMC_OK;
    rc = eval_rows(h, nullptr, nullptr, nslots, nslots, nullptr, h->cfg.precision, h->d_rates, h->d_R, h->d_E);
    if (rc != AKMC_OK) return rc;
    CK(h, cudaStreamSynchronize(h->stream));
    rc = harvest_events(h);
    if (rc != AKMC_OK) return rc;
    rc = check_overflow(h, "akmc_rates");
    if (rc != AKMC_OK) return rc;
    std::vector<double> R((size_t)nslots * 8), E((size_t)nslots * 8);
    CK(h, cudaMemcpy(R.data(), h->d_rates, R.size() * sizeof(double), cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(E.data(), h->d_E, E.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < vr.size(); ++i)
        for (int k = 0; k < 8; ++k) {
            if (rates_out) rates_out[i * 8 + k] = R[(size_t)vr[i].slot * 8 + k];
            if (barriers_out) barriers_out[i * 8 + k] = E[(size_t)vr[i].slot * 8 + k];
        }
    return AKMC_OK;
}

int akmc_eval_windows(akmc_handle* h, const uint8_t* windows, int64_t n, int32_t precision, double* E_out)
{
    if (!h) return AKMC_ERR_RUNTIME;
    if (n < 0 || n > (1 << 26) || !windows || !E_out) return fail(h, AKMC_ERR_INVALID, "bad window batch");
    if (precision != AKMC_PREC_FP64 && precision != AKMC_PREC_FP32 && precision != AKMC_PREC_FP16_FAST)
        return fail(h, AKMC_ERR_INVALID, "unknown precision");
    for (int64_t i = 0; i < n * kWin; ++i)
        if (windows[i] > kVac) return fail(h, AKMC_ERR_INVALID, "species code > 6 in window");
    if (n == 0) return AKMC_OK;
    uint8_t* d_w = nullptr;
    double* d_e = nullptr;
    CK(h, pool_malloc(&d_w, (size_t)n * kWin));
    CK(h, pool_malloc(&d_e, (size_t)n * 8 * sizeof(double)));
    CK(h, cudaMemcpy(d_w, windows, (size_t)n * kWin, cudaMemcpyHostToDevice));
    int rc = eval_rows(h, nullptr, nullptr, (int)n, (int)n, d_w, precision, nullptr, nullptr, d_e);
    if (rc == AKMC_OK) {
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess) e = cudaMemcpy(E_out, d_e, (size_t)n * 8 * sizeof(double), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = fail(h, AKMC_ERR_CUDA, std::string("eval_windows: ") + cudaGetErrorString(e));
        else rc = harvest_events(h);
        if (rc == AKMC_OK) rc = check_overflow(h, "akmc_eval_windows");
    }
    cudaFree(d_w);
    cudaFree(d_e);
    return rc;
}

void akmc_free(akmc_handle* h)
{
    if (!h) return;
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->xchg_n)
        std::fprintf(stderr, "[akmc exchange] %lld exchanges: pack %.2f us, unpack incl. wait for the peers %.2f us per "
                     "exchange\n", (long long)h->xchg_n, 1e3 * h->xchg_ms[0] / h->xchg_n, 1e3 * h->xchg_ms[1] / h->xchg_n);
    if (h->d_phase_cycles) {
        static unsigned long long c[kDiagWords];
        std::memset(c, 0, sizeof(c));
        cudaMemcpy(c, h->d_phase_cycles, sizeof(c), cudaMemcpyDeviceToHost);
        const double t = c[7] ? (double)c[7] : 1.0;
        if (c[7])
            std::fprintf(stderr, "[akmc phase timing] tiles=%llu cycles/tile: gather %.0f encode %.0f M1 %.0f E1 %.0f M2 %.0f"
                         " E2 %.0f M3+E3 %.0f; CTA loop %.0f cycles x %llu CTAs\n", c[7], c[0] / t, c[1] / t, c[2] / t,
                         c[3] / t, c[4] / t, c[5] / t, c[6] / t, c[9] ? (double)c[8] / (double)c[9] : 0.0, c[9]);
        const unsigned long long* d = c + 32;
        if (d[7]) {
            const double n = (double)d[7];
            std::fprintf(stderr, "[akmc engine] CTA-launches=%llu (phase %llu) iterations/CTA %.1f (max %llu) rounds/CTA %.1f"
                         " eval-rounds/CTA %.1f refills/CTA %.1f; cycles/CTA: control %.0f rounds %.0f select %.0f total %.0f\n",
                         d[7], d[10], d[0] / n, d[1], d[2] / n, d[3] / n, d[8] / n, d[4] / n, d[5] / n, d[6] / n, d[9] / n);
            if (d[40] || d[46])
                std::fprintf(stderr, "[akmc engine-tc] per CTA: rounds %.1f (with rows %.1f) group-iterations %.1f refills %.1f;"
                             " evaluator cycles: exchange %.0f L2+E2 %.0f L3+partials %.0f E3 %.0f | control cycles: wait %.0f"
                             " select %.0f refill %.0f rows+gather %.0f L1 %.0f\n", d[40] / n, d[41] / n, d[51] / n, d[52] / n,
                             d[42] / n, d[43] / n, d[44] / n, d[45] / n, d[46] / n, d[47] / n, d[48] / n, d[49] / n, d[50] / n);
            std::fprintf(stderr, "[akmc engine] cycles/CTA: refill %.0f rows %.0f gather+memo %.0f | L1 %.0f exchange %.0f"
                         " (k>0 rounds %.0f) L2+E2 %.0f L3+partials %.0f E3 %.0f\n", d[11] / n, d[12] / n, d[13] / n,
                         d[14] / n, d[15] / n, d[19] / n, d[16] / n, d[17] / n, d[18] / n);
            if (d[29]) std::fprintf(stderr, "[akmc engine] memo-hit chain: %llu events of %llu checks (%.1f per CTA-launch)\n", d[29], d[30], d[29] / n);
            if (d[90])
                std::fprintf(stderr, "[akmc overlap] %llu phases: boundary list published %.1f us after the engine start "
                             "(%llu before it); engine %.1f us\n", d[90], 1e-3 * d[88] / d[90], d[91], 1e-3 * d[89] / d[90]);
            if (d[56] + d[57] + d[58])
                std::fprintf(stderr, "[akmc engine] dataflow refill cycles/CTA: candidates %.0f readiness %.0f activation %.0f\n",
                             d[56] / n, d[57] / n, d[58] / n);
            std::fprintf(stderr, "[akmc engine] L1 split: memo move %.0f layer 1 %.0f async fences + barrier %.0f\n",
                         d[20] / n, d[21] / n, d[22] / n);
            if (d[24] + d[25] + d[26] + d[27])
                std::fprintf(stderr, "[akmc engine] layer-1 probe (warp 0): index %.0f b1 %.0f loads+adds %.0f store %.0f\n",
                             d[24] / n, d[25] / n, d[26] / n, d[27] / n);
        }
        {
            const unsigned long long* b = c + 128 + 512 + 64;
            if (b[4] && b[8] && b[12]) {
                const double T = (double)b[8];           // tiles (all CTAs)
                const double P = 4.0 * (double)b[4] / (double)b[12];   // producer warps per CTA (4 epilogue warps)
                std::fprintf(stderr, "[akmc bulk] tiles %.0f; cycles per tile -- producer warp (%.0f): gather %.0f wait-A %.0f "
                             "layer-1 %.0f wait-meta %.0f | MMA thread: wait-A %.0f wait-TMEM %.0f issue %.0f | epilogue "
                             "warp: wait %.0f E2+L3 %.0f E3 %.0f\n", T, P, b[0] / (P * T), b[1] / (P * T), b[2] / (P * T),
                             b[3] / (P * T), b[5] / T, b[6] / T, b[7] / T, b[9] / (4 * T), b[10] / (4 * T), b[11] / (4 * T));
            }
        }
        // per-iteration trace: iteration index -> CTA count, mean rows / misses / running domains, cycles
        const unsigned long long* tr = c + 128;
        if (tr[0]) {
            std::fprintf(stderr, "[akmc iter trace] it: ctas rows miss run | cyc ctl rounds sel | rounds\n");
            for (int i = 0; i < 64; ++i) {
                const unsigned long long* t = tr + 8 * i;
                if (!t[0]) continue;
                const double n = (double)t[0];
                std::fprintf(stderr, "[akmc iter trace] %2d: %6llu %6.1f %6.1f %6.1f | %7.0f %7.0f %7.0f | %.2f\n", i, t[0],
                             t[1] / n, t[2] / n, t[3] / n, t[4] / n, t[5] / n, t[6] / n, t[7] / n);
            }
            std::fprintf(stderr, "[akmc iter trace] iterations per CTA launch:");
            for (int i = 0; i < 64; ++i)
                if (c[128 + 512 + i]) std::fprintf(stderr, " %d:%llu", i, c[128 + 512 + i]);
            std::fprintf(stderr, "\n");
        }
        cudaFree(h->d_phase_cycles);
        h->d_phase_cycles = nullptr;
    }
    free_all(h);
    delete h;
}

} // extern "C"
