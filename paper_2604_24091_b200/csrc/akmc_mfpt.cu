// akmc_mfpt.cu -- exact mean-first-passage-time solver (sec. V.A.3, Eqs. 5-6;
// S:265-305).  On an enumerated state space the MFPT tau(s) to the absorbing set solves the Poisson equation
// by Dynkin's formula,  sum_a Gamma_a(s) [tau(Phi(s,a)) - tau(s)] + 1 = 0,  tau = 0 on absorbing states, i.e.
// the M-matrix system (D - R) tau = 1 with D = diag(Gamma_tot) and R the transient-to-transient rates.  It is the
// exact time reference of the world model's learned increment (Eq. 7 plug-in identity).
//
// Solver: BiCGSTAB with Jacobi preconditioning as ONE cooperative launch over the whole GPU (grid-stride loops,
// grid-wide barriers between the dependent steps, no host round trip per iteration).  Every reduction has a
// fixed order -- per-thread partials over a fixed index set, a fixed block tree, block partials summed in block
// order by every block -- so a solve is deterministic for a given launch shape (it sums in another order than
// a single-CTA solve would: the result is Eq. 5's to the solver tolerance, not bit-identical across shapes).
#include <algorithm>
#include <cmath>
#include <cooperative_groups.h>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>

#include "../../include/akmc.h"

namespace cg = cooperative_groups;

namespace {

constexpr int kMT = 256;                 // threads per block
constexpr int kMaxBlocks = 1024;

struct MfptParams {
    const int64_t* rp;
    const int32_t* col;
    const double* rate;
    int64_t n;
    double tol;
    int max_iter;
    double* x;          // tau
    double* r; double* rh; double* p; double* v; double* s; double* t; double* y; double* z; double* dinv;
    double* part;       // [3][kMaxBlocks] block partials
    double* out;        // [0] relative residual, [1] iterations
};

// fixed-order reduction of up to 3 per-thread values over the grid; every block returns the same sums
__device__ void grid_sum3(const MfptParams& P, cg::grid_group& g, double a, double b, double c, double* res, int k)
{
    __shared__ double red[3][kMT / 32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double v[3] = {a, b, c};
    for (int q = 0; q < k; ++q) {
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
        if (lane == 0) red[q][w] = v[q];
    }
    __syncthreads();
    if (tid < k) {
        double u = 0.0;
        for (int i = 0; i < kMT / 32; ++i) u += red[tid][i];
        P.part[tid * kMaxBlocks + blockIdx.x] = u;
    }
    g.sync();
    for (int q = 0; q < k; ++q) {
        double u = 0.0;
        for (int i = 0; i < (int)gridDim.x; ++i) u += P.part[q * kMaxBlocks + i];
        res[q] = u;
    }
    g.sync();                                    // the partials are reused by the next reduction
}

// y = A x with A = D - R (rows: diagonal = sum of all outgoing rates, off-diagonal = -rate to transient cols)
__device__ void spmv(const MfptParams& P, const double* x, double* yv)
{
    for (int64_t i = blockIdx.x * (int64_t)kMT + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * kMT) {
        double diag = 0.0, off = 0.0;
        for (int64_t e = P.rp[i]; e < P.rp[i + 1]; ++e) {
            const double g = P.rate[e];
            diag += g;
            const int32_t c = P.col[e];
            if (c >= 0) off = fma(g, x[c], off);
        }
        yv[i] = fma(diag, x[i], -off);
    }
}

#define GRID_FOR(i) for (int64_t i = blockIdx.x * (int64_t)kMT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kMT)

__global__ void __launch_bounds__(kMT) mfpt_bicgstab_kernel(const MfptParams P)
{
    cg::grid_group g = cg::this_grid();
    const int64_t n = P.n;
    double red[3];
    // Jacobi preconditioner, x0 = D^-1 1, r = 1 - A x0
    GRID_FOR(i) {
        double d = 0.0;
        for (int64_t e = P.rp[i]; e < P.rp[i + 1]; ++e) d += P.rate[e];
        P.dinv[i] = 1.0 / d;
        P.x[i] = P.dinv[i];
    }
    g.sync();
    spmv(P, P.x, P.t);
    g.sync();
    double loc = 0.0;
    GRID_FOR(i) {
        const double ri = 1.0 - P.t[i];
        P.r[i] = ri; P.rh[i] = ri; P.p[i] = 0.0; P.v[i] = 0.0;
        loc += ri * ri;
    }
    grid_sum3(P, g, loc, 0.0, 0.0, red, 1);
    const double bnorm = sqrt((double)n);
    double rnorm = sqrt(red[0]);
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    int it = 0;
    while (it < P.max_iter && rnorm > P.tol * bnorm) {
        ++it;
        loc = 0.0;
        GRID_FOR(i) loc += P.rh[i] * P.r[i];
        grid_sum3(P, g, loc, 0.0, 0.0, red, 1);
        const double rho1 = red[0];
        if (rho1 == 0.0) break;
        const double beta = (rho1 / rho) * (alpha / omega);
        rho = rho1;
        GRID_FOR(i) {
            P.p[i] = P.r[i] + beta * (P.p[i] - omega * P.v[i]);
            P.y[i] = P.dinv[i] * P.p[i];
        }
        g.sync();
        spmv(P, P.y, P.v);
        loc = 0.0;
        GRID_FOR(i) loc += P.rh[i] * P.v[i];                 // (own rows of v: written by this thread above)
        grid_sum3(P, g, loc, 0.0, 0.0, red, 1);
        const double rv = red[0];
        if (rv == 0.0) break;
        alpha = rho / rv;
        GRID_FOR(i) {
            P.s[i] = P.r[i] - alpha * P.v[i];
            P.z[i] = P.dinv[i] * P.s[i];
        }
        g.sync();
        spmv(P, P.z, P.t);
        double ts = 0.0, tt = 0.0;
        GRID_FOR(i) { ts += P.t[i] * P.s[i]; tt += P.t[i] * P.t[i]; }
        grid_sum3(P, g, ts, tt, 0.0, red, 2);
        omega = red[1] > 0.0 ? red[0] / red[1] : 0.0;
        loc = 0.0;
        GRID_FOR(i) {
            P.x[i] += alpha * P.y[i] + omega * P.z[i];
            const double ri = P.s[i] - omega * P.t[i];
            P.r[i] = ri;
            loc += ri * ri;
        }
        grid_sum3(P, g, loc, 0.0, 0.0, red, 1);
        rnorm = sqrt(red[0]);
        if (omega == 0.0) break;
    }
    // true residual of Eq. 5 with the final tau
    g.sync();
    spmv(P, P.x, P.t);
    loc = 0.0;
    GRID_FOR(i) { const double ri = 1.0 - P.t[i]; loc += ri * ri; }
    grid_sum3(P, g, loc, 0.0, 0.0, red, 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) { P.out[0] = sqrt(red[0]) / bnorm; P.out[1] = (double)it; }
}

} // namespace

extern "C" int akmc_mfpt_solve(const int64_t* row_ptr, const int32_t* col, const double* rate, int64_t n, double tol,
                               int32_t max_iter, double* tau_out, int32_t* iters_out, double* resid_out)
{
    if (n <= 0 || !row_ptr || !col || !rate || !tau_out || !(tol > 0.0) || max_iter < 1) return AKMC_ERR_INVALID;
    if (row_ptr[0] != 0) return AKMC_ERR_INVALID;
    const int64_t nnz = row_ptr[n];
    for (int64_t i = 0; i < n; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) return AKMC_ERR_INVALID;
        double d = 0.0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            if (!(rate[e] >= 0.0) || !std::isfinite(rate[e]) || col[e] < -1 || col[e] >= n) return AKMC_ERR_INVALID;
            d += rate[e];
        }
        if (!(d > 0.0)) return AKMC_ERR_INVALID;        // a transient state needs an outgoing event
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return AKMC_ERR_CUDA;
    int64_t* d_rp = nullptr; int32_t* d_col = nullptr; double* d_rate = nullptr; double* d_vec = nullptr;
    cudaError_t e = cudaMalloc(&d_rp, (size_t)(n + 1) * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc(&d_col, (size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d_rate, (size_t)std::max<int64_t>(nnz, 1) * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&d_vec, ((size_t)10 * n + 2 + 3 * kMaxBlocks) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(d_rp, row_ptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(d_col, col, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(d_rate, rate, (size_t)nnz * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        MfptParams P{};
        P.rp = d_rp; P.col = d_col; P.rate = d_rate; P.n = n; P.tol = tol; P.max_iter = max_iter;
        double* b = d_vec;
        P.x = b; P.r = b + n; P.rh = b + 2 * n; P.p = b + 3 * n; P.v = b + 4 * n; P.s = b + 5 * n; P.t = b + 6 * n;
        P.y = b + 7 * n; P.z = b + 8 * n; P.dinv = b + 9 * n; P.out = b + 10 * n; P.part = b + 10 * n + 2;
        // grid: co-resident blocks (cooperative launch), ~4 rows per thread at least
        int nsm = 0, per_sm = 0;
        e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mfpt_bicgstab_kernel, kMT, 0);
        if (e == cudaSuccess) {
            const int64_t want = (n + 4 * kMT - 1) / (4 * kMT);
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)nsm * std::min(per_sm, 2),
                                                                          (int64_t)kMaxBlocks}));
            void* args[] = {&P};
            e = cudaLaunchCooperativeKernel((void*)mfpt_bicgstab_kernel, dim3(grid), dim3(kMT), args, 0, nullptr);
        }
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        double out[2] = {0.0, 0.0};
        if (e == cudaSuccess) e = cudaMemcpy(tau_out, P.x, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(out, P.out, sizeof(out), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) {
            if (iters_out) *iters_out = (int32_t)out[1];
            if (resid_out) *resid_out = out[0];
        }
    }
    cudaFree(d_rp); cudaFree(d_col); cudaFree(d_rate); cudaFree(d_vec);
    return e == cudaSuccess ? AKMC_OK : AKMC_ERR_CUDA;
}
