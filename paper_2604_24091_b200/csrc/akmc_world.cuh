// akmc_world.cuh -- interface of the world-model time mode kernel (akmc_world.cu).
#pragma once
#include "akmc_kernels.cuh"

namespace akmc {

constexpr int kWorldMaxVac = 64;        // vacancies per voxel in world-model mode (one CTA holds a voxel)
constexpr int kWorldMaxHidden = 256;    // Poisson-time network hidden width

struct WorldParams {
    uint8_t* species;
    int4* vac;
    Frame F;
    GeomTables G;
    PhysParams P;           // pair-KRA tables (physical rates -> Gamma_tot of Eq. 7) and per-voxel kT
    const double* mlp;      // FP64 network weights; raw outputs = policy logits (Eq. 1)
    const double* tnet;     // Poisson-time net: Wt1[448*H], bt1[H], wt2[H], bt2[1] (FP64)
    int H;
    double tau_act;         // Eq. 1 temperature
    int nvox;
    const int* vstart;      // [nvox + 1] slot ranges per voxel
    int n_events;           // events per voxel in this launch
    long long* nev;         // per-voxel event counters (Philox counter, A16)
    int* term;              // per-voxel terminal flags
    double* clock;          // per-voxel clocks (advanced by Eq. 7)
    uint64_t seed;
    DevCounters* ctr;
};

size_t world_smem_bytes();
cudaError_t world_setup();
cudaError_t launch_world(const WorldParams& p, int num_sms, cudaStream_t s);

} // namespace akmc
