// akmc_world.cu -- world-model time mode: the paper's own simulation step
// (sec. V.A.1, sec. V.A.3), in serial / voxel-batch mode, FP64.
//
// Per voxel (one competing set, A15) and event:
//   policy   z_{i,k} = the barrier network's raw outputs read as logits; Eq. 1: zhat = z / tau_act for
//            admissible hops, -inf (weight 0) for masked ones; Eq. 2: global softmax over the voxel's
//            concatenated logits -> (i, k) drawn with probability exp(zhat) / sum exp(zhat), realised as the
//            canonical tree + descent over the weights det_exp(min(zhat, 700)) (reading W1) with the serial
//            Philox counter (A16);
//   time     Eq. 7: dtau_hat = (uhat(s) - Gamma_tot(s)/Gamma_tot(s') uhat(s')) / Gamma_tot(s), Gamma_tot from the
//            physical pair-KRA rates, uhat = softplus(Poisson-time MLP(mean one-hot window over
//            the voxel's vacancies)); clock += max(dtau_hat, 1e-3 / Gamma_tot(s)) (W4).
// Every FP64 operation follows the oracle's order (oracle/akmc_oracle.c orc_run_world), so trajectories and
// clocks are bit-exact.  One CTA (256 threads) per voxel; a vacancy is re-evaluated only when its 64-byte
// window changed (exact: the logits and rates are pure functions of the window, R7).
#include "akmc_kernels.cuh"
#include "akmc_world.cuh"

namespace akmc {
namespace {

constexpr int kWT = 256;

__device__ __forceinline__ double softplus_dev(double y)
{
    if (y > 0.0) return __dadd_rn(y, det_log(__dadd_rn(1.0, det_exp(-y))));
    return det_log(__dadd_rn(1.0, det_exp(y)));
}

__device__ __forceinline__ double dtau_hat_dev(double u_s, double g_s, double u_sp, double g_sp)
{
    if (!(g_sp > 0.0)) return __ddiv_rn(u_s, g_s);
    return __ddiv_rn(__dsub_rn(u_s, __dmul_rn(__ddiv_rn(g_s, g_sp), u_sp)), g_s);
}

struct WorldSmem {
    uint8_t win[kWorldMaxVac][kWin];      // current windows of the voxel's vacancies
    uint8_t cached[kWorldMaxVac][kWin];   // windows of the cached evaluations
    double W[kWorldMaxVac][8];            // policy weights
    double G[kWorldMaxVac][8];            // physical rates
    double Rw[4 * kWorldMaxVac + 8];      // policy tree
    double Rg[4 * kWorldMaxVac + 8];      // physical-rate tree
    double h1[kHid], h2[kHid], z[8];
    double hp[kHid];                      // Poisson-net hidden layer
    int cnt[448];
    double xf[448];                       // pooled Poisson-net input count_f / m
    int4 pos[kWorldMaxVac];
    int slot[kWorldMaxVac];
    int dirty[kWorldMaxVac];
    double wtot, gtot, uhat;
    int P, nlev;
};

// evaluate the voxel's state: windows, (re)evaluate dirty rows, trees, uhat
__device__ void world_eval(const WorldParams& p, WorldSmem& S, int m, int vox, unsigned long long& rows)
{
    const int tid = threadIdx.x;
    // windows of all members (thread = (member, slot)); dirty = window differs from the cached evaluation
    for (int t = tid; t < m * kWin; t += kWT) {
        const int a = t / kWin, j = t % kWin;
        // plain coherent load: this kernel writes the lattice
        S.win[a][j] = p.species[neighbour_site(p.F, S.pos[a], p.G.off[j][0], p.G.off[j][1], p.G.off[j][2])];
    }
    if (tid < m) S.dirty[tid] = 0;
    __syncthreads();
    for (int t = tid; t < m * kWin; t += kWT) {
        const int a = t / kWin, j = t % kWin;
        if (S.win[a][j] != S.cached[a][j]) S.dirty[a] = 1;
    }
    __syncthreads();
    // Poisson-time network input on the pooled windows (counts of the 448 one-hot features, x_f = count_f / m, each
    // quotient formed once -- the same division the oracle does per use): it needs only the windows, so its hidden
    // chains can run beside the barrier network's last stage below
    for (int f = tid; f < 448; f += kWT) S.cnt[f] = 0;
    __syncthreads();
    for (int t = tid; t < m * kWin; t += kWT) {
        const int a = t / kWin, j = t % kWin;
        atomicAdd(&S.cnt[kSpecies * j + S.win[a][j]], 1);
    }
    __syncthreads();
    for (int f = tid; f < 448; f += kWT) S.xf[f] = __ddiv_rn((double)S.cnt[f], (double)m);
    int last_dirty = -1;
    for (int a = 0; a < m; ++a) if (S.dirty[a]) last_dirty = a;       // (block-uniform: shared flags)
    __syncthreads();
    // the Poisson net's hidden unit j: one sequential fma chain over f (the oracle's order); threads 32 .. 32 + H
    // (beside the last dirty row's layer 3 / rates on threads 0-7), else after the rows on threads 0 .. H
    auto poisson_hidden = [&](int j) {
        double acc = p.tnet[448 * (size_t)p.H + j];                    // bt1
#pragma unroll 32
        for (int f = 0; f < 448; ++f) acc = __fma_rn(S.xf[f], p.tnet[(size_t)f * p.H + j], acc);
        S.hp[j] = acc > 0.0 ? acc : 0.0;
    };
    const bool pois_beside = last_dirty >= 0 && p.H <= kWT - 32;
    const double* W1 = p.mlp;
    const double* b1 = W1 + 448 * kHid;
    const double* W2 = b1 + kHid;
    const double* b2 = W2 + kHid * kHid;
    const double* W3 = b2 + kHid;
    const double* b3 = W3 + kHid * 8;
    for (int a = 0; a < m; ++a) {
        if (!S.dirty[a]) continue;                      // block-uniform (shared flag after a barrier)
        ++rows;                                         // a network row actually evaluated (R4 mlp_rows)
        // (loops unrolled so that many weight loads are in flight ahead of the sequential FP64 chain: the sums keep
        // the oracle's order, bit for bit)
        const int j = tid;
        double acc = b1[j];
#pragma unroll 32
        for (int s = 0; s < kWin; ++s) acc = __dadd_rn(acc, W1[(size_t)(kSpecies * s + S.win[a][s]) * kHid + j]);
        S.h1[j] = acc > 0.0 ? acc : 0.0;
        __syncthreads();
        acc = b2[j];
#pragma unroll 32
        for (int i = 0; i < kHid; ++i) acc = __fma_rn(S.h1[i], W2[(size_t)i * kHid + j], acc);
        S.h2[j] = acc > 0.0 ? acc : 0.0;
        __syncthreads();
        if (j < 8) {
            acc = b3[j];
#pragma unroll 32
            for (int i = 0; i < kHid; ++i) acc = __fma_rn(S.h2[i], W3[i * 8 + j], acc);
            // Eq. 1 mask and temperature on the raw output (the policy logit, no clamp); physical pair-KRA rate
            double w = 0.0, g = 0.0;
            if (S.win[a][j] != (uint8_t)kVac) {
                double zh = __ddiv_rn(acc, p.tau_act);
                if (zh > 700.0) zh = 700.0;
                w = det_exp(zh);
                double E = 0.0;
                pair_barrier(S.win[a], j, p.G, p.P, E);
                g = arrhenius(E, p.P, vox);
            }
            S.W[a][j] = w;
            S.G[a][j] = g;
        } else if (pois_beside && a == last_dirty && tid >= 32 && tid < 32 + p.H) {
            poisson_hidden(tid - 32);
        }
        if (j < kWin) S.cached[a][j] = S.win[a][j];
        __syncthreads();
    }
    if (!pois_beside) {
        if (tid < p.H) poisson_hidden(tid);
        __syncthreads();
    }
    // serial tail, two threads of different warps at once: uhat (thread 0); member sums and trees (thread 32)
    if (tid == 0) {
        const double* wt2 = p.tnet + 448 * (size_t)p.H + p.H;
        double y = wt2[p.H];                                           // bt2
        for (int j = 0; j < p.H; ++j) y = __fma_rn(S.hp[j], wt2[j], y);
        S.uhat = m > 0 ? softplus_dev(y) : 0.0;
    } else if (tid == 32) {
        // per-member sums in hop order, then the canonical trees (A17); Rw keeps the policy tree
        for (int a = 0; a < m; ++a) {
            double sw = 0.0, sg = 0.0;
            for (int k = 0; k < 8; ++k) { sw = __dadd_rn(sw, S.W[a][k]); sg = __dadd_rn(sg, S.G[a][k]); }
            S.Rw[a] = sw;
            S.Rg[a] = sg;
        }
        int P = 1, nlev = 0;
        S.gtot = m > 0 ? tree_build(S.Rg, m, P, nlev) : 0.0;
        S.wtot = m > 0 ? tree_build(S.Rw, m, P, nlev) : 0.0;
        S.P = P; S.nlev = nlev;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kWT) world_serial_kernel(const __grid_constant__ WorldParams p)
{
    extern __shared__ __align__(16) uint8_t wsm[];
    WorldSmem& S = *reinterpret_cast<WorldSmem*>(wsm);
    const int tid = threadIdx.x;
    unsigned long long events = 0, evals = 0, terminal = 0, rows = 0;
    for (int v = blockIdx.x; v < p.nvox; v += gridDim.x) {
        const int s0 = p.vstart[v], m = p.vstart[v + 1] - s0;
        if (tid < m) { S.slot[tid] = s0 + tid; S.pos[tid] = p.vac[s0 + tid]; }
        for (int t = tid; t < m * kWin; t += kWT) S.cached[t / kWin][t % kWin] = 0xFF;   // nothing cached
        __syncthreads();
        if (p.term[v]) continue;                       // a terminal voxel stays frozen
        world_eval(p, S, m, v, rows);
        for (int e = 0; e < p.n_events; ++e) {
            evals += 8ull * (unsigned long long)m;
            if (!(S.wtot > 0.0) || !(S.gtot > 0.0)) {   // no feasible event
                if (tid == 0) p.term[v] = 1;
                terminal += 1;
                break;
            }
            if (tid == 0) {
                const unsigned long long n = (unsigned long long)p.nev[v];
                double u_sel, u_t;
                philox_uniforms(p.seed, make_uint4((uint32_t)n, (uint32_t)(n >> 32), (uint32_t)v, 0u), u_sel, u_t);
                double r = __dmul_rn(u_sel, S.wtot);
                const int a = tree_descend(S.Rw, m, S.P, S.nlev, r);
                const int k = pick_hop(S.W[a], r);
                const int4 ov = S.pos[a];
                int4 nv = ov;
                nv.y = wrap2(ov.y + p.G.off[k][0], 2 * p.F.L[0]);
                nv.z = wrap2(ov.z + p.G.off[k][1], 2 * p.F.L[1]);
                nv.w = wrap2(ov.w + p.G.off[k][2], 2 * p.F.L[2]);
                const uint8_t tn = S.win[a][k];        // the target's species (window slot k, 1NN)
                write_site(p.species, p.F, ov.x, ov.y, ov.z, ov.w, tn);
                write_site(p.species, p.F, nv.x, nv.y, nv.z, nv.w, (uint8_t)kVac);
                S.pos[a] = nv;
                p.vac[S.slot[a]] = nv;
            }
            __threadfence_block();
            __syncthreads();
            const double u_s = S.uhat, g_s = S.gtot;
            world_eval(p, S, m, v, rows);              // s' (also the next event's s)
            if (tid == 0) {
                const double dt = dtau_hat_dev(u_s, g_s, S.uhat, S.gtot);
                const double fl = __ddiv_rn(1e-3, g_s);
                p.clock[v] = __dadd_rn(p.clock[v], dt > fl ? dt : fl);
                p.nev[v] += 1;
            }
            events += 1;
            __syncthreads();
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (events) atomicAdd(&p.ctr->events, events);
        if (evals) atomicAdd(&p.ctr->hop_evals, evals);
        if (terminal) atomicAdd(&p.ctr->terminal, terminal);
        if (rows) atomicAdd(&p.ctr->mrows, rows);
    }
}

} // namespace

size_t world_smem_bytes() { return sizeof(WorldSmem); }

cudaError_t world_setup()
{
    return cudaFuncSetAttribute(world_serial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(WorldSmem));
}

cudaError_t launch_world(const WorldParams& p, int num_sms, cudaStream_t s)
{
    const int grid = std::max(1, std::min(p.nvox, num_sms * 4));
    world_serial_kernel<<<grid, kWT, sizeof(WorldSmem), s>>>(p);
    return cudaGetLastError();
}

} // namespace akmc
