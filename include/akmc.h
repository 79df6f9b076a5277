/*
 * akmc.h -- C-ABI of the B200-native AKMC vacancy-hop step (AtomWorld, arXiv 2604.24091).
 *
 * The library (paper_2604_24091_b200/lib/libakmc.so) runs the data-parallel hot path of the
 * paper's atomistic world model on one B200 per process: for every vacancy it gathers the
 * 64-site neighbourhood (sec. V.A.1, sec. VI.C), evaluates the barrier network
 * (sec. V.B.1) or the pair KRA model, turns barriers
 * into Arrhenius rates (Eq. 8), and selects/applies one hop per competing set with a
 * residence-time draw (Eq. 2 read as BKL) from Philox4x32-10.
 * Citations: P:NNN = PAPER.md line, S:NNN = SPEC.md line, A<n> = reading n in DESIGN.md sec. 3.
 *
 * Conventions common to every call
 *  - All pointers passed IN are caller-owned HOST memory, copied before the call returns.
 *    *_out buffers are caller-allocated host memory.  The handle owns all device memory.
 *  - One handle per process and GPU (the device current at akmc_init).  Calls on one handle are
 *    not reentrant.  Every call is synchronous: it returns after its device work completes.
 *  - Return value: AKMC_OK or an AKMC_* status.  On a non-OK status, akmc_last_error() gives a
 *    one-line message; the state is unchanged for AKMC_ERR_INVALID and AKMC_TERMINAL.
 *  - Site index (canonical, per voxel): i = 2*(x + Lx*(y + Ly*z)) + b, basis b in {0,1};
 *    a multi-voxel lattice is n_voxels such blocks back to back (global site = voxel*sites + i).
 *  - Species codes (A6): Fe 0, Cu 1, Ni 2, Mn 3, Si 4, P 5, vacancy 6; n_species must be 7.
 *  - Vacancy slot ids: the vacancies present at akmc_init, ordered by global site index; a
 *    slot keeps its identity as the vacancy moves.
 *  - Determinism: within one precision mode, equal (config, inputs, seed) give equal output
 *    bits for any launch configuration.  In AKMC_PREC_FP64 mode the trajectory is bit-equal to
 *    the FP64 CPU oracle (oracle/akmc_oracle.c) -- DESIGN.md sec. 5 fixes every FP operation.
 */
#ifndef AKMC_H
#define AKMC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (categories follow SPEC cli exit codes S:724-725, terminal signal S:199) */
enum {
    AKMC_OK = 0,
    AKMC_ERR_RUNTIME = 1,   /* internal error (bad handle, exceeded capacity)            */
    AKMC_ERR_INVALID = 2,   /* invalid configuration or inputs (list at akmc_init)       */
    AKMC_TERMINAL = 3,      /* no feasible event in a competing set       */
    AKMC_ERR_CUDA = 4,      /* CUDA runtime error / no device / missing sm_100a          */
    AKMC_ERR_NCCL = 5       /* NCCL error (multi-GPU)                                    */
};

enum { AKMC_MODEL_PAIR = 0, AKMC_MODEL_MLP = 1 };
/* precision of the barrier evaluation (the selection is always FP64, A17):
 *  FP64 : sequential fma in the oracle's order + det_exp -> bit-exact trajectories
 *  FP32 : "matrix multiplication ... executed in FP32": layer 1 FP64-accumulated sparse
 *         embedding bag rounded to FP32; layer 2 on tcgen05 tensor cores as an FP32-equivalent
 *         3-pass fp16 split (hi*hi + hi*lo + lo*hi, FP32 accumulate in TMEM); layer 3 FP32.
 *         Per-hop rates within 1e-5 relative of FP64 (north star).  Pair model: same as FP64.
 * FP16_FAST : SURVEY 8(b) "fast" mode, for information only: layers 2-3 as ONE fp16 pass (hi parts only,
 *         FP32 accumulate; 1/3 of the tensor-core work and half the h1 traffic).  Rates ~1e-3 relative:
 *         it does NOT meet the 1e-5 bar; trajectories are valid AKMC at approximate rates.  MLP only. */
enum { AKMC_PREC_FP64 = 0, AKMC_PREC_FP32 = 1, AKMC_PREC_FP16_FAST = 2 };

typedef struct akmc_config {
    int32_t  cells[3];        /* Lx,Ly,Lz bcc cells per voxel; each even, >= 4 and <= 4096   */
    int32_t  n_voxels;        /* >= 1 independent periodic voxels                          */
    int32_t  n_species;       /* must be 7 (A6); vacancy code 6                                    */
    int32_t  barrier_model;   /* AKMC_MODEL_PAIR or AKMC_MODEL_MLP        */
    int32_t  precision;       /* AKMC_PREC_FP64, AKMC_PREC_FP32 or AKMC_PREC_FP16_FAST             */
    int32_t  domain_cells[3]; /* sublattice domain edge (reading A19/A21): {0,0,0} => serial BKL,  */
                              /* one competing set per voxel (A15); else each even, >= 6, divides */
                              /* cells (sector = domain/2 >= 3 cells, A20)                          */
    double   temperature_K;   /* > 0                                                       */
    double   nu0;             /* attempt frequency, > 0                                    */
    double   kB;              /* Boltzmann constant eV/K; passed so both sides share bits  */
    double   window_s;        /* Delta_win per phase (A22); > 0 in sublattice mode                 */
    uint64_t seed;            /* Philox key (A16)                                                  */
    int32_t  gpu_grid[3];     /* spatial decomposition over ranks (C5): the global lattice  */
                              /* is gpu_grid x cells; rank r owns block (r%gx, r/gx%gy, r/(gx*gy)).      */
                              /* {1,1,1} for a single rank.  world > 1 requires sublattice mode and      */
                              /* n_voxels == 1; axes with gpu_grid == 1 stay periodic inside the block.  */
    int32_t  rank, world;     /* this process's rank / world size; world must equal prod(gpu_grid)     */
    uint8_t  nccl_id[128];    /* ncclUniqueId from akmc_nccl_unique_id() on rank 0, broadcast by the    */
                              /* caller (e.g. torch.distributed); ignored when world == 1               */
} akmc_config;

typedef struct akmc_counters {
    int64_t events;           /* hops applied                                                      */
    int64_t hop_evals;        /* 8 x vacancy evaluations (masked hops included), S:587 accounting  */
    int64_t iterations;       /* inner iterations (serial: events per voxel; sublattice: a8 loops) */
    int64_t clamps;           /* pair-model barriers clamped at 0 (A12)                            */
    int64_t terminal_voxels;  /* competing sets that hit Gamma_tot == 0 (serial mode)              */
    int64_t sweeps;           /* sublattice sweeps completed since init                            */
    int64_t kernel_launches;  /* kernels launched by the library                                   */
    int64_t mlp_launches;     /* launches of the dominant (barrier) kernel                         */
    int64_t mlp_rows;         /* vacancy rows evaluated by it                                      */
    double  mlp_ms;           /* its summed CUDA-event time (only when profiling is enabled)       */
    double  wall_ms;          /* host wall time inside akmc_step                                    */
} akmc_counters;

typedef struct akmc_handle akmc_handle;

/* Create a simulation on the current CUDA device.
 *  species : n_voxels * 2*Lx*Ly*Lz bytes, canonical order (see above).
 *  eps     : [2][7][7] pair energies eV, eps[s][a][b] (s = 1NN, 2NN), symmetric;
 *            required for AKMC_MODEL_PAIR, ignored (may be NULL) for the MLP.
 *  E0      : [7] base barriers eV; required for the pair model.
 *  mlp     : FP64 weights W1[448*256] (row f = 7*slot + species), b1[256], W2[256*256]
 *            (row = input), b2[256], W3[256*8], b3[8]; required for AKMC_MODEL_MLP.
 * AKMC_ERR_INVALID when: a cell count is odd or < 4; n_voxels < 1; n_species != 7; a species code
 * > 6; vacancies exceed 1% of sites; T, nu0 or kB <= 0; domains do not divide the lattice
 * or a sector is < 3 cells; window_s <= 0 in sublattice mode; world != prod(gpu_grid) or world != 1;
 * eps not symmetric; a NaN/Inf in eps, E0 or mlp; an unknown model or precision.
 * AKMC_ERR_CUDA when no CUDA device is present or the device is not sm_100.                       */
int akmc_init(const akmc_config* cfg, const uint8_t* species, const double* eps, const double* E0,
              const double* mlp, akmc_handle** out);

/* Advance: serial mode -> n events per voxel; sublattice mode -> n sweeps of 8
 * phases (reading A19).  ctr (optional) receives the counters accumulated over this
 * call.  Returns AKMC_TERMINAL when some competing set had no feasible event (its state is left
 * unchanged from that point); other voxels still advance. */
int akmc_step(akmc_handle* h, int64_t n, akmc_counters* ctr);

/* Voxel-ensemble mode (voxels evolved independently to a common physical time; serial mode
 * only): every voxel runs BKL events until its next event would happen after t_end_s, or
 * max_events events of this call, or Gamma_tot == 0.  The draw whose event time clock + dt exceeds
 * t_end_s is discarded and its Philox counter (the voxel's event index) is not consumed, so splitting a
 * run at any horizons gives the trajectory of the unsplit run; voxel clocks stay at their last event
 * (raw AKMC time, <= t_end_s).  Voxels run concurrently in one persistent engine launch (each CTA pulls
 * voxels as slots free up).  Returns like akmc_step; AKMC_ERR_INVALID in sublattice mode, for a
 * non-finite t_end_s or max_events outside [0, 2^30] (one launch per call), and when the legacy
 * (non-engine) serial path is active.                                                                   */
int akmc_run_until(akmc_handle* h, double t_end_s, int64_t max_events, akmc_counters* ctr);

/* Read back the state.  species_out: n_voxels*sites bytes (may be NULL); vac_sites_out: global
 * site index of each vacancy slot (may be NULL) with *n_vac_inout = capacity in / count out
 * (a short buffer returns AKMC_ERR_INVALID without writing); clock_s_out: [n_voxels] simulated
 * seconds (may be NULL); ctr_out: counters accumulated since init (may be NULL).              */
int akmc_state(akmc_handle* h, uint8_t* species_out, int64_t* vac_sites_out, int64_t* n_vac_inout,
               double* clock_s_out, akmc_counters* ctr_out);

/* Vacancies currently owned by this rank (multi-rank: vacancies migrate between blocks): global slot
 * ids (gid_out, may be NULL) and global canonical site indices over the global lattice (site_out, may
 * be NULL), sorted by gid; *n_inout = capacity in / count out.                                     */
int akmc_vacancies(akmc_handle* h, int64_t* gid_out, int64_t* site_out, int64_t* n_inout);

/* Dataflow sweeps (the asynchronous sublattice with readiness signals; S:526-529,
 * S:572-580), single-rank sublattice handles: instead of 8 phases separated by grid-wide boundaries, one engine
 * launch per sweep in which each tile of domains starts phase q as soon as the 27 tiles around it have finished
 * phase q-1 (a domain's phase-q reads and writes stay inside its 26 neighbour domains, reading A20), so the tail
 * of one phase overlaps the next.  The trajectory is the synchronous sweep's, bit for bit (same Philox counters,
 * same per-domain order).  on = 0 returns to phase-synchronous launches.  AKMC_ERR_INVALID for serial or
 * multi-rank handles or the legacy loop; a capacity overflow during a sweep (more than 64 vacancies entering one
 * tile in a sweep) makes that akmc_step return AKMC_ERR_RUNTIME.                                              */
int akmc_set_dataflow(akmc_handle* h, int32_t on);

/* Multi-rank exchange statistics (C5): out3[0] = per-phase exchanges done, out3[1] = messages this
 * rank sent (direct exchange: one per distinct peer and phase; AKMC_EXCHANGE=shift: the paper's shift
 * communication, P:420-427, 2 per decomposed axis -- 1 when two ranks share the axis), out3[2] = bytes sent.  */
int akmc_exchange_stats(akmc_handle* h, int64_t* out3);

/* Dynamic voxel scheduling (sec. V.C.2, Eq. 10), serial / voxel-batch handles: voxels are
 * dispatched to the persistent engine's slots in descending workload proxy W_v = M_v exp(-E_v / (kB T_v)),
 * M_v = 8 x the voxel's vacancies, E_v = the composition-weighted mean base barrier E0 of its atoms (0 without
 * pair parameters), T_v its temperature (akmc_set_voxel_temperatures recomputes the order); ties keep voxel
 * order.  The order changes no trajectory, only the makespan of batches larger than the resident slots.
 * order_out [n_voxels] receives the voxel ids in dispatch order.  AKMC_ERR_INVALID in sublattice mode.     */
int akmc_voxel_order(akmc_handle* h, int32_t* order_out);

/* World-model time mode (sec. V.A.1 Eqs. 1-2, sec. V.A.3 Eq. 7;
 * S:356-409).  Serial / voxel-batch handles with barrier_model AKMC_MODEL_MLP at AKMC_PREC_FP64 whose akmc_init
 * got eps and E0.  After this call every akmc_step(n) event of a voxel: (1) reads the network's raw outputs
 * as policy logits z_{i,k}; Eq. 1 masks infeasible hops (weight 0) and divides by tau_act; Eq. 2's softmax over
 * the voxel's concatenated logits selects (i, k) (weights det_exp(min(z/tau, 700)), canonical tree + descent,
 * the serial Philox counter); (2) applies the hop; (3) advances the voxel clock by max(dtau_hat, 1e-3 /
 * Gamma_tot(s)) with Eq. 7 dtau_hat = (uhat(s) - Gamma_tot(s)/Gamma_tot(s') uhat(s')) / Gamma_tot(s), Gamma_tot
 * = total pair-KRA rate and uhat = softplus of the Poisson-time network on the mean one-hot window
 * of the voxel's vacancies.  tnet: host FP64 Wt1[448*hidden] (row f = 7*slot + species), bt1[hidden],
 * wt2[hidden], bt2[1], copied.  A voxel with no feasible event (or Gamma_tot = 0) is terminal.  FP64
 * throughout: trajectories and clocks are bit-equal to the oracle's orc_run_world.  AKMC_ERR_INVALID (state
 * unchanged) for a sublattice handle, another model/precision, missing eps/E0, hidden outside [1, 256],
 * tau_act <= 0, non-finite weights, or more than 64 vacancies in a voxel.  akmc_run_until is not available
 * in this mode.                                                                                          */
int akmc_set_world_model(akmc_handle* h, const double* tnet, int32_t hidden, double tau_act);

/* Exact MFPT solver (sec. V.A.3 Eq. 5): tau on the transient states
 * of an enumerated state space from  sum_a Gamma_a(s) [tau(Phi(s,a)) - tau(s)] + 1 = 0,  tau = 0 on the
 * absorbing set (no handle; runs on the current CUDA device).  Transitions of transient state i are
 * row_ptr[i] .. row_ptr[i+1]-1 (host, row_ptr[0] = 0): target col[e] (a transient index, or -1 = into the
 * absorbing set) with rate rate[e] >= 0 s^-1; every transient state needs a positive total rate.  tau_out [n]
 * (host, seconds).  Jacobi-preconditioned BiCGSTAB until ||1 - A tau|| <= tol ||1|| or max_iter iterations;
 * iters_out / resid_out (may be NULL) report the iterations and the final relative residual of Eq. 5.  The
 * exact u = Gamma_tot tau it yields is the reference of the world model's Eq. 7 (plug-in identity).
 * AKMC_ERR_INVALID for n <= 0, bad CSR, negative / non-finite rates, a state with no outgoing rate, tol <= 0
 * or max_iter < 1; AKMC_ERR_CUDA on a device error.                                                         */
int akmc_mfpt_solve(const int64_t* row_ptr, const int32_t* col, const double* rate, int64_t n, double tol,
                    int32_t max_iter, double* tau_out, int32_t* iters_out, double* resid_out);

/* Checkpoint / resume (lattice + vacancy list + clock + counters is a full checkpoint; the
 * counter-based RNG needs no state).  akmc_progress reads the rest of the run position: nev_out [n_voxels]
 * (may be NULL) = each voxel's serial event index (the Philox counter of its next event, S:195-198 / A16),
 * sweep_out (may be NULL) = sublattice sweeps done (the next sweep's sector permutation and phase counters).
 * akmc_restore, on a handle freshly created by akmc_init from a checkpointed lattice, re-establishes that
 * position: vac_sites [n_vac] (may be NULL) = the checkpoint's vacancy sites in SLOT order (akmc_state's
 * vac_sites_out), which fixes the slot ids and therefore every competing-set tree order (A17); clock_s
 * [n_voxels] and nev [n_voxels] may be NULL; sweep >= 0.  The resumed run is bit-identical to the unsplit
 * one.  AKMC_ERR_INVALID (state unchanged) when vac_sites is not a permutation of the lattice's vacancy
 * sites, slots are not grouped by voxel in ascending order, a clock is negative or non-finite, a counter is
 * negative, or the handle is multi-rank (world > 1).                                                     */
int akmc_progress(akmc_handle* h, int64_t* nev_out, int64_t* sweep_out);
int akmc_restore(akmc_handle* h, const int64_t* vac_sites, int64_t n_vac, const double* clock_s, const int64_t* nev,
                 int64_t sweep);

/* Diagnostics: the voxel-0 block INCLUDING its halo, cells [-2, L+2) per axis, canonical order
 * (2*(x + (Lx+4)*(y + (Ly+4)*z)) + b over the extended box); out holds 2*(Lx+4)*(Ly+4)*(Lz+4) bytes.  */
int akmc_debug_extended(akmc_handle* h, uint8_t* out);

/* Write a fresh ncclUniqueId (128 bytes) for akmc_config.nccl_id (call on rank 0 only). */
int akmc_nccl_unique_id(uint8_t* out128);

/* Per-hop rates of the current state in the handle's precision, [n_vac][8] slot order, masked
 * hops exactly 0; barriers_out (may be NULL) gets the barriers E [n_vac][8] eV.    */
int akmc_rates(akmc_handle* h, double* rates_out, double* barriers_out);

/* Diagnostics: evaluate the barrier model on n caller-given windows (host [n][64] species bytes in
 * window-slot order) at the given precision; E_out [n][8] barriers in eV
 * (mask not applied).  Uses the handle's weights/parameters; state untouched.                   */
int akmc_eval_windows(akmc_handle* h, const uint8_t* windows, int64_t n, int32_t precision, double* E_out);

/* Per-voxel temperature (SURVEY 8(d) C4 variant "per-voxel T uniform in 558-577 K"; the voxels
 * of a mesoscopic model see different local conditions).  T_K: host [n] Kelvin, n == n_voxels, each
 * finite and > 0, copied.  Every later rate of a vacancy in voxel v is nu0 exp(-E/(kB*T_v))
 * (Eq. 8) with kB*T_v formed as one IEEE product, as for the uniform T; the barrier memo is cleared
 * (its rates were formed at the old T).  akmc_eval_windows keeps the configured temperature_K.
 * Callable between steps in any mode; AKMC_ERR_INVALID on a wrong n or a bad T (state unchanged). */
int akmc_set_voxel_temperatures(akmc_handle* h, const double* T_K, int32_t n);

/* Diagnostics (no handle; current device): the device's deterministic exp / log (DESIGN.md sec. 5.3,
 * reading A29) on n host doubles x -> y.  fn 0 = det_exp (rates, Eq. 8), 1 = det_log (residence time,
 * S:198).  AKMC_ERR_INVALID for another fn or bad pointers, AKMC_ERR_CUDA on a device error.       */
int akmc_debug_math(int32_t fn, const double* x, int64_t n, double* y);

/* Launch the library's kernels on this CUDA stream (cudaStream_t as void*; NULL = the handle's
 * own stream).  profile != 0 records CUDA events around every barrier-kernel launch (mlp_ms).  */
int akmc_set_stream(akmc_handle* h, void* stream);
int akmc_set_profiling(akmc_handle* h, int32_t profile);

void akmc_free(akmc_handle* h);

/* Message of the last non-OK status on this handle (or of the last failed akmc_init when h is
 * NULL).  Never NULL; "" when there was no error.                                              */
const char* akmc_last_error(const akmc_handle* h);

/* Library version string, e.g. "akmc-b200 0.1 sm_100a". */
const char* akmc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AKMC_H */
