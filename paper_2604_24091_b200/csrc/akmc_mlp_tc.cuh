// akmc_mlp_tc.cuh -- interface of the tcgen05 barrier-network kernel (FP32-equivalent mode).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "akmc_device.cuh"

namespace akmc {

constexpr int kTileM = 128;          // rows (vacancies) per CTA tile = TMEM lanes
constexpr int kKChunk = 16;          // K per pipeline stage (one UMMA K-step)
constexpr int kNChunks = kHid / kKChunk;
constexpr int kStages = 4;
constexpr int kSplitBytes = kHid * kKChunk * 2;        // one fp16 split of a B chunk: 8 KiB
constexpr int kStageBytes = 2 * kSplitBytes;           // hi + lo: 16 KiB
constexpr int kABytes = kTileM * kHid * 2;             // one fp16 split of the A tile: 64 KiB
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
    const double* W1p;               // [448][256] Fe-referenced layer-1 rows (fp64)
    const double* b1p;               // [256] layer-1 bias + sum of Fe rows (fp64)
    const __half* Bimg;              // [kNChunks][2][kSplitBytes/2] W2^T splits in UMMA smem image
    const float* b2;                 // [256]
    const float* W3;                 // [256][8]
    const float* b3;                 // [8]
    float w2_unscale;                // 2^-sb (W2 was scaled by 2^sb before splitting)
    PhysParams P;
    // outputs indexed by slot (or by window index)
    double* rates;                   // [.][8] or nullptr
    double* Rsum;                    // [.]    or nullptr
    double* E;                       // [.][8] or nullptr
    unsigned long long* overflow;    // count of |h1| beyond the fp16 range (diagnostic)
};

// smem bytes needed by the kernel
size_t mlp_tc_smem_bytes();
// persistent launch: min(num_sms, ceil(max_rows/128)) CTAs loop over the tiles of the device row count
cudaError_t launch_mlp_tc(const MlpTcParams& p, int max_rows, int num_sms, cudaStream_t s);
// one-time attribute setup (max dynamic smem)
cudaError_t mlp_tc_setup();

} // namespace akmc
