// akmc_engine.cuh -- the sublattice phase engine: a persistent, cluster-resident kernel that runs every
// domain of a sublattice phase to the end of its time window with no grid-wide synchronisation.
//
// Why: in the windowed synchronous sublattice scheme (reading A19) the inner loop
// of a phase runs until the LAST domain overshoots the window, and the per-domain event count has a
// heavy tail (a vacancy next to a low-barrier solute flickers thousands of times per window).  A
// grid-synchronous inner loop pays one full barrier-network latency per event of the slowest domain.
// Here every CTA owns a handful of domains and iterates them independently; the 8 CTAs of a cluster
// share one barrier-network evaluator whose weights stay resident in shared memory (each CTA holds a
// 64-column slice of W2 and the matching 64 rows of W3), and results are memoised per vacancy (exact: the rates are a pure
// function of the 64-byte window).
#pragma once
#include "akmc_kernels.cuh"

namespace akmc {

constexpr int kClusterN = 4;                   // CTAs per cluster; CTA r owns hidden columns [64r, 64r+64)
constexpr int kSliceN = kHid / kClusterN;      // 64
constexpr int kRoundRows = 128 / kClusterN;    // rows a CTA contributes per evaluation round (tile M = 128)
constexpr int kSlots = 128;                    // domain slots per CTA (a domain with > 2 vacancies spans several)
constexpr int kSlotCap = 2;                    // vacancies per slot
constexpr int kRowCap = kSlots * kSlotCap;     // vacancies a CTA holds at once (128)
constexpr int kW1Rows = 1 + (kSpecies - 1) * kWin;   // b1' then W1'(s, slot) rows: 385
constexpr int kMyTiles = 32;                   // dataflow: tiles per CTA (tiles are dealt round-robin)
constexpr int kArrCap = 64;                    // dataflow: arrivals per tile and sweep

// exact memo of the barrier network per vacancy slot (2 ways, most recent first)
struct MemoEntry {
    uint8_t key[kWin];      // window bytes (0xFF: empty -- species codes are < kSpecies)
    double G[8];            // rates
    double R;               // sum in hop order
    int clamps;             // pair-model clamps of this evaluation (kept so counters match the oracle)
    int pad;
};
static_assert(sizeof(MemoEntry) == 144, "memo entry layout");
static_assert(sizeof(MemoEntry) == kMemoBytes && offsetof(MemoEntry, R) == kMemoROff, "memo layout seen by segments_kernel");

struct EngineWeights {
    const float* W1f;       // [385][256] FP32: row 0 = b1' = b1 + sum_slot W1[slot,Fe]; row 1+(s-1)*64+slot = W1'
    const uint8_t* W2img;   // [4 CTAs][16 K-steps][hi 2 KiB | lo 2 KiB] fp16 UMMA images of W2^T column slices * 2^s2
    const double* W3d;      // [256][8] FP64 W3 (CTA r of a cluster loads rows [64r, 64r+64)); layer 3 runs in FP64
    const float* b2;        // [256]
    const double* b3;       // [8]
    float s2u;              // 2^(t1-s2): undoes the W2 image scale 2^s2 and the h1 scale 2^-t1
    float h1s;              // 2^-t1: power-of-two activation scale chosen at init from weight bounds so that
                            // |h1| * 2^-t1 <= 2^15 for every window (the fp16 hi part cannot overflow)
    const double* mlp64;    // FP64 weights (verify precision)
};

enum EngineMode { kEnginePhase = 0, kEngineEval = 1 };

struct EngineParams {
    int mode;               // kEnginePhase: run the phase's domains; kEngineEval: evaluate a row list
    int model;              // AKMC_MODEL_PAIR (0) / AKMC_MODEL_MLP (1)
    int fast;               // 1: AKMC_PREC_FP16_FAST -- single-pass fp16 layers 2-3 (hi parts only)
    uint8_t* species;
    int4* vac;
    Frame F;
    GeomTables G;
    PhysParams P;
    SubParams S;
    const PhaseInfo* ph;
    const Segment* segs;
    const int* members;
    const int4* mpos;       // member positions at phase start (parallel to members)
    DevCounters* ctr;
    MemoEntry* memo;        // [vcap][2] (phase mode) or nullptr
    double* scratch;        // trees of segments with > 16 members (4 doubles per member, by member offset)
    int* iscratch;
    // eval mode
    const uint8_t* windows; // [n][64] or nullptr (then rows -> vac slots, gathered)
    const int* rows;        // slot list or nullptr (row i = slot i)
    const int* nrows_dev;   // device row count or nullptr
    int nrows_host;
    unsigned int* cursor;   // work cursor (eval mode), zeroed before launch
    double* rates;          // [.][8] outputs (eval mode)
    double* Rsum;
    double* E;
    EngineWeights W;
    uint8_t* stage;         // [clusters][4 CTAs][hi | lo] h1 rows staged in L2 for the multicast
    uint8_t* wstore;        // [CTAs][kRowCap][64] full windows of the rows a CTA holds
    // serial / voxel-batch mode (a10): a "domain" is a whole voxel, each runs n_events BKL events per launch
    int serial;             // 1: segments = voxels, no window/sector; 0: sublattice phase
    int nseg_host;          // serial: number of voxels (segments)
    int n_events;           // serial: events per voxel in this launch
    long long* nev;         // serial: per-voxel event counters (Philox counter, P:294-298 / S:195-203)
    int* term;              // serial: per-voxel terminal flags
    double* clock;          // serial: per-voxel clocks
    int seg_cap;            // phase: > 0 -> hot segments at segs[0, nhot), cold ones at segs[seg_cap-1-i]
    int overlap;            // multi-rank: 1 -> segs holds the interior domains; the boundary ones follow in segs2
    const Segment* segs2;   //   once ctr->bready == ph->phase + 1 (published by a stream-parallel kernel)
    int horizon;            // serial: 1 -> a voxel also stops at its first draw with clock + dt > t_end
    double t_end;           //   (akmc_run_until; the draw is discarded, its counter not consumed)
    // dataflow sweep (f1, P:405-418 readiness signals; single rank): one launch runs the 8 phases of a sweep; a
    // tile of domains starts phase q once the 27 tiles around it have finished phase q-1 (akmc_engine.cu)
    int df;                 // 1: dataflow sweep
    int ntiles;             // tiles in all voxels
    int tdom[3];            // domains per tile edge
    int NT[3];              // tiles per axis per voxel
    long long* done_phase;  // [ntiles] last finished global phase (release / acquire)
    const int* tile_off;    // [ntiles + 1] base member offsets (vacancies in the tile at sweep start)
    const int* tile_mem;    // base member slots
    int* arr_cnt;           // [ntiles] vacancies that entered the tile during the sweep
    int* arr_slot;          // [ntiles][kArrCap]
    int ring_cap;           // per-CTA capacity of the activation ring (members / positions / keys)
    int* ring_slot;         // [CTAs][ring_cap]
    int4* ring_pos;
    unsigned long long* ring_key;
    int* df_err;            // capacity overflows (arrivals, ring) -> AKMC_ERR_RUNTIME
    unsigned long long* overflow;   // fp16 range clamps / capacity overflows (diagnostic, must stay 0)
    unsigned long long* diag;       // [16] optional timing/iteration diagnostics (AKMC_PHASE_TIMING)
    int* watch;             // optional [CTAs][8] progress words in mapped host memory (AKMC_WATCHDOG)
};

// bulk evaluator (akmc_bulk.cu): the same per-row arithmetic on many rows, one persistent CTA per SM
struct BulkParams {
    const uint8_t* species;
    const int4* vac;
    Frame F;
    GeomTables G;
    PhysParams P;
    const uint8_t* windows; // [n][64] or nullptr (then rows -> vac slots, gathered)
    const int* rows;        // slot list or nullptr (row i = slot i)
    const int* nrows_dev;   // device row count or nullptr
    int nrows_host;
    EngineWeights W;
    const uint8_t* W2full;  // [16 K-steps][hi 8 KiB | lo 8 KiB] fp16 UMMA images of W2^T (N = 256) * 2^s2
    double* rates;          // [.][8] or nullptr
    double* Rsum;
    double* E;
    unsigned long long* overflow;
    int fast;
    unsigned long long* diag;   // optional [16] per-role cycle sums (AKMC_PHASE_TIMING)
};
cudaError_t bulk_setup();
cudaError_t launch_bulk(const BulkParams& p, int max_rows, int num_sms, cudaStream_t s);

// dataflow sweep: base lists of the tiles (cnt / cursor scratch [ntiles], off [ntiles + 1], mem [vcap])
cudaError_t launch_df_prep(const EngineParams& p, const int4* vac, int nv, int* cnt, int* off, int* cursor, int* mem,
                           cudaStream_t s);
size_t engine_smem_bytes();
cudaError_t engine_setup();
// clusters of 8 that can be co-resident (persistent grid); 0 on failure
int engine_max_clusters();
// tc = 1: FP32-equivalent tensor-core evaluator (cluster launch); tc = 0: FP64 evaluator (plain launch)
cudaError_t launch_engine(const EngineParams& p, bool tc, int nclusters, int num_sms, cudaStream_t s);

} // namespace akmc
