// akmc_p2p.cuh -- the default per-phase exchange of the C5 decomposition: deltas stored
// straight into the peers' mailboxes over NVLink (CUDA IPC), tagged so that no system-scope fence is needed, and
// (overlap) arrivals activated into the next phase's boundary domain lists.  Split from akmc_dist.cuh because
// the activation needs the sublattice types of akmc_kernels.cuh.
#pragma once
#include "akmc_kernels.cuh"

namespace akmc {

// ---------------------------------------------------------------- per-phase exchange over NVLink peer memory
// Each rank owns a mailbox [npeer][2 parities][cap + 1] x 16 B; peer r's deltas for exchange e land in r's region
// of our mailbox (parity e & 1), written by r's pack kernel with plain 64-bit stores through the CUDA IPC mapping.
// Every 64-bit word carries the exchange's tag (the low 32 bits of e), so the receiver needs no ordering from the
// sender: it polls the region's header word (count | tag << 32) and then each entry's two words until their tags
// read e -- a 64-bit store is seen whole or not at all, and a stale word from exchange e - 2 carries another tag.
// The sender issues no system-scope fence (each one waits for an NVLink round trip): its only ordering is the
// device-scope handshake that lets the last block write the counts.  Two parities suffice: a peer can write
// exchange e + 2 only after it has received our exchange e + 1, which we send after our unpack of e.
constexpr int kP2PBlocks = 16;         // the per-phase log is ~0.3-10 K entries: a few blocks
struct PeerBoxes {
    int4* box[kMaxPeers];                  // our region (parity 0) in peer r's mailbox; parity 1 at + cap + 1
    unsigned long long* flag[kMaxPeers];   // (unused by the tagged protocol; kept for the mapping's layout)
    int* cnt;                              // [npeer] local allocation counters of this exchange
    unsigned int* done;                    // blocks of the pack kernel that have finished (last block publishes)
    unsigned long long* ep;                // exchanges completed on this rank (device-side, so that the exchange
};                                         // can live inside a replayed CUDA graph): exchange e = *ep + 1

__device__ __forceinline__ void st_relaxed_sys_u64(void* p, unsigned long long v)
{
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int kExchangeTimeout = 1 << 30;  // flag bit in the exchange overflow word

// entry (global half-cell coordinates < 2^16, value w) <-> two tagged words
__device__ __forceinline__ void put_entry(int4* dst, int g0, int g1, int g2, int w, uint32_t tag)
{
    unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
    st_relaxed_sys_u64(d, (unsigned long long)(uint32_t)g0 | ((unsigned long long)(uint32_t)g1 << 16) |
                              ((unsigned long long)(uint32_t)g2 << 32) | ((unsigned long long)(tag & 0xFFFFu) << 48));
    st_relaxed_sys_u64(d + 1, (unsigned long long)(uint32_t)w | ((unsigned long long)tag << 32));
}

__device__ __forceinline__ void pack_p2p(const int4* __restrict__ log, unsigned long long* nlog_p, int logcap, const Frame& F,
                                         const DistParams& D, const uint8_t* __restrict__ species, const PeerBoxes& B,
                                         unsigned long long epoch, int* overflow)
{   // (epoch = *B.ep + 1, read by the caller before any block can complete the exchange)
    const int n = (int)min((unsigned long long)logcap, *nlog_p);
    const size_t par = (size_t)(epoch & 1ull) * (size_t)(D.cap + 1);
    const uint32_t tag = (uint32_t)epoch;
    const int lane = threadIdx.x & 31;
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    if (blockIdx.x == 0 && threadIdx.x == 0 && *nlog_p > (unsigned long long)logcap) atomicAdd(overflow, 1);
    // block-uniform trip count, so that every lane of a warp takes part in the per-peer ballots: one counter
    // atomic per warp and peer instead of one per entry
    for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
        const int i = i0 + (int)threadIdx.x;
        const bool have = i < n;
        int4 e = make_int4(0, 0, 0, 0);
        int gc[3] = {0, 0, 0}, gp[3] = {0, 0, 0};
        if (have) {
            e = log[i];
            if (e.w < kMigrateBase) e.w = species[site_of(F, 0, e.x, e.y, e.z)];   // the site's FINAL value
            const int p[3] = {e.x, e.y, e.z};
            for (int a = 0; a < 3; ++a) {
                gc[a] = imod((p[a] >> 1) + D.O[a], D.G[a]);
                gp[a] = 2 * gc[a] + (p[a] & 1);
            }
        }
        for (int r = 0; r < D.npeer; ++r) {
            const bool want = have && ((e.w >= kMigrateBase) ? in_block(gc, D.peerO[r], F, D)
                                                             : in_extended(gc, D.peerO[r], F, D));
            const unsigned m = __ballot_sync(0xffffffffu, want);
            if (!m) continue;
            const int leader = __ffs(m) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&B.cnt[r], __popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (want) {
                const int k = base + __popc(m & lt);
                if (k < D.cap) put_entry(&B.box[r][par + 1 + k], gp[0], gp[1], gp[2], e.w, tag);   // NVLink stores
                else atomicAdd(overflow, 1);
            }
        }
    }
    // the last block to finish publishes the counts (device-scope handshake on the reservation counters)
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(B.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        if (threadIdx.x == 0) __threadfence();
        __syncthreads();
        const int r = threadIdx.x;
        if (r < D.npeer) {
            const int c = min(atomicAdd(&B.cnt[r], 0), D.cap);
            st_relaxed_sys_u64(&B.box[r][par], (unsigned long long)(uint32_t)c | ((unsigned long long)tag << 32));
            B.cnt[r] = 0;
        }
        if (r == 0) { *B.done = 0u; *nlog_p = 0ull; }
    }
}
static __global__ void pack_p2p_kernel(const int4* __restrict__ log, unsigned long long* nlog_p, int logcap, Frame F,
                                       DistParams D, const uint8_t* __restrict__ species, PeerBoxes B, int* overflow)
{
    pack_p2p(log, nlog_p, logcap, F, D, species, B, *(volatile unsigned long long*)B.ep + 1, overflow);
}

// wait for every peer's deltas of exchange `epoch` (tags), then apply them (same semantics as unpack_deltas_kernel)
// act (overlap, optional): arrivals join the next phase's domain lists as activate_kernel would have put them
struct ArrivalActivation {
    const PhaseInfo* ph;   // the next phase, or nullptr (no activation)
    SubParams S;
    int* dmin;
    int* head;
    int* next;
    long long* bdom;       // boundary domains holding active vacancies (appended: first member of a domain)
    DevCounters* ctr;
};
__device__ __forceinline__ void unpack_p2p(const int4* __restrict__ mbox, unsigned long long epoch, const Frame& F,
                                           const DistParams& D, uint8_t* species, int4* vac, int* gid, int* nvac_local,
                                           int vcap, const FreeList& FL, int* overflow, const ArrivalActivation& act,
                                           unsigned long long* ep)
{
    const int nfree0 = *(volatile int*)&FL.cnt[0];
    const uint32_t tag = (uint32_t)epoch;
    const size_t par = (size_t)(epoch & 1ull) * (size_t)(D.cap + 1);
    // bounded waits: a peer that never publishes (a crashed or diverged rank) must not hang the GPU -- after 30 s
    // the exchange is abandoned and reported (kExchangeTimeout in the overflow word -> AKMC_ERR_RUNTIME)
    __shared__ int cnt_s[kMaxPeers];
    if (threadIdx.x < D.npeer) {
        const int4* hdr = mbox + (size_t)threadIdx.x * 2 * (D.cap + 1) + par;
        const unsigned long long t0 = globaltimer_ns();
        unsigned long long h;
        while ((uint32_t)((h = ld_relaxed_sys_u64(hdr)) >> 32) != tag) {
            __nanosleep(32);
            if (globaltimer_ns() - t0 > 30000000000ull) { atomicOr(overflow, kExchangeTimeout); h = 0; break; }
        }
        cnt_s[threadIdx.x] = min((int)(uint32_t)h, D.cap);
    }
    __syncthreads();
    for (int r = 0; r < D.npeer; ++r) {
        const int4* buf = mbox + (size_t)r * 2 * (D.cap + 1) + par;
        const int cnt = cnt_s[r];
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&buf[1 + i]);
            unsigned long long a, b;
            const unsigned long long t0 = globaltimer_ns();
            bool arrived = true;
            for (;;) {
                a = ld_relaxed_sys_u64(src);
                b = ld_relaxed_sys_u64(src + 1);
                if ((uint32_t)(b >> 32) == tag && (uint32_t)(a >> 48) == (tag & 0xFFFFu)) break;
                if (globaltimer_ns() - t0 > 30000000000ull) { atomicOr(overflow, kExchangeTimeout); arrived = false; break; }
            }
            if (!arrived) continue;                      // (reported; a stale word is never applied)
            const int gp[3] = {(int)(a & 0xFFFFu), (int)((a >> 16) & 0xFFFFu), (int)((a >> 32) & 0xFFFFu)};
            const int w = (int)(uint32_t)b;
            int lp[3];
            bool ok = true;
            for (int ax = 0; ax < 3; ++ax) {
                if (F.wrap[ax]) { lp[ax] = gp[ax]; continue; }
                int d = imod(gp[ax] - 2 * D.O[ax], 2 * D.G[ax]);
                if (d >= 2 * (F.L[ax] + kHalo)) d -= 2 * D.G[ax];
                lp[ax] = d;
                if (d < -2 * kHalo || d >= 2 * (F.L[ax] + kHalo)) ok = false;
            }
            if (!ok) { atomicAdd(overflow, 1); continue; }
            if (w >= kMigrateBase) {
                const int slot = arrival_slot(FL, nfree0, nvac_local);
                if (slot < vcap) {
                    const int4 nv = make_int4(0, lp[0], lp[1], lp[2]);
                    vac[slot] = nv;
                    gid[slot] = w - kMigrateBase;
                    if (act.ph) {
                        long long dd; int sec;
                        dom_sector(nv, act.S, dd, sec);
                        if (sec == act.ph->sector) {
                            atomicMin(&act.dmin[dd], w - kMigrateBase);
                            const int prev = atomicExch(&act.head[dd], slot);
                            act.next[slot] = prev;
                            if (prev < 0) act.bdom[atomicAdd(&act.ctr->nbdom, 1ull)] = dd;   // (an arrival: boundary)
                        }
                    }
                } else {
                    atomicAdd(overflow, 1);
                }
            } else {
                write_site(species, F, 0, lp[0], lp[1], lp[2], (uint8_t)w);
            }
        }
    }
    unpack_done(FL, nfree0, ep, epoch);
}
static __global__ void unpack_p2p_kernel(const int4* __restrict__ mbox, unsigned long long* ep, Frame F, DistParams D,
                                         uint8_t* species, int4* vac, int* gid, int* nvac_local, int vcap, FreeList FL,
                                         int* overflow, ArrivalActivation act = ArrivalActivation{})
{
    unpack_p2p(mbox, *(volatile unsigned long long*)ep + 1, F, D, species, vac, gid, nvac_local, vcap, FL, overflow, act, ep);
}
// send and receive of one exchange in one launch (the unoverlapped per-phase path): every block packs its share,
// the last one publishes the counts, then every block waits for the peers' deltas and applies its share
static __global__ void exchange_p2p_kernel(const int4* __restrict__ log, unsigned long long* nlog_p, int logcap, Frame F,
                                           DistParams D, PeerBoxes B, const int4* __restrict__ mbox,
                                           uint8_t* species, int4* vac, int* gid, int* nvac_local, int vcap, FreeList FL,
                                           int* overflow)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");                // (PDL: the phase's engine has completed)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the next activation may become resident
    const unsigned long long epoch = *(volatile unsigned long long*)B.ep + 1;   // (raised by the last block at the end)
    pack_p2p(log, nlog_p, logcap, F, D, species, B, epoch, overflow);
    __syncthreads();
    unpack_p2p(mbox, epoch, F, D, species, vac, gid, nvac_local, vcap, FL, overflow, ArrivalActivation{}, B.ep);
}

} // namespace akmc
