// akmc_mlp_tc.cuh -- interface of the tcgen05 barrier-network kernel (FP32-equivalent mode).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "akmc_device.cuh"

namespace akmc {

constexpr int kTileM = 128;                    // rows (vacancies) per CTA tile = TMEM lanes
constexpr int kK1 = 16 + kWin * (kSpecies - 1);   // layer-1 K: bias K-step + one-hot over 6 non-Fe species = 400
constexpr int kKChunk = 16;                    // K per ring stage (one UMMA K-step)
constexpr int kChunksL1 = kK1 / kKChunk;       // 25 (chunk 0 = bias, then species-major groups of 16 slots)
constexpr int kChunksL2 = kHid / kKChunk;      // 16
constexpr int kChunksTile = kChunksL1 + kChunksL2;   // 41 image chunks (W1' then W2)
constexpr int kStages = 4;
constexpr int kSplitBytes = kHid * kKChunk * 2;        // one fp16 split of a B chunk (N = 256): 8 KiB
constexpr int kStageBytes = 2 * kSplitBytes;           // hi + lo: 16 KiB
constexpr int kABytes = kTileM * kHid * 2;             // one fp16 split of the A tile (K = 256): 64 KiB
constexpr int kN3 = 16;                                // layer-3 N padded from 8 to the UMMA minimum
constexpr int kW3SplitBytes = kN3 * kHid * 2;          // 8 KiB
constexpr float kLoScale = 2048.0f;                    // lo parts are stored * 2^11

struct MlpTcParams {
    // window source: either (species, vac) with the geometry tables, or explicit windows
    const uint8_t* species;
    const int4* vac;
    const uint8_t* windows;          // [n][64] or nullptr
    Frame F;
    GeomTables G;
    const int* rows;                 // slot ids to evaluate (nullptr => row i = slot i)
    const int* nrows_dev;            // device row count (nullptr => nrows_host)
    int nrows_host;
    // weights (prepared at init)
    const __half* Bimg;              // [41][2][N=256 x K=16] bias + W1'^T (25 chunks) then W2^T (16), UMMA images
    const __half* W3img;             // [2][N=16 x K=256] W3^T splits, UMMA image
    const float* b2;                 // [256]
    const double* b3;                // [8]
    float s1_unscale;                // 2^-s1 (W1' scaled by 2^s1 before splitting)
    float s2_unscale;                // 2^-s2
    double s3_unscale;               // 2^-s3
    PhysParams P;
    // outputs indexed by slot (or by window index)
    double* rates;                   // [.][8] or nullptr
    double* Rsum;                    // [.]    or nullptr
    double* E;                       // [.][8] or nullptr
    unsigned long long* overflow;    // count of |h| beyond the fp16 range (diagnostic)
    unsigned long long* phase_cycles; // [10] optional: summed clock64 per tile phase (AKMC_PHASE_TIMING)
};

// smem bytes needed by the kernel
size_t mlp_tc_smem_bytes();
// persistent launch: min(num_sms, ceil(max_rows/128)) CTAs loop over the tiles of the device row count
cudaError_t launch_mlp_tc(const MlpTcParams& p, int max_rows, int num_sms, cudaStream_t s);
// one-time attribute setup (max dynamic smem)
cudaError_t mlp_tc_setup();

} // namespace akmc
