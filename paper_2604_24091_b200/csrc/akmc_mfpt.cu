// akmc_mfpt.cu -- exact mean-first-passage-time solver (sec. V.A.3, Eqs. 5-6;
// S:265-305).  On an enumerated state space the MFPT tau(s) to the absorbing set solves the Poisson equation
// by Dynkin's formula,  sum_a Gamma_a(s) [tau(Phi(s,a)) - tau(s)] + 1 = 0,  tau = 0 on absorbing states, i.e.
// the M-matrix system (D - R) tau = 1 with D = diag(Gamma_tot) and R the transient-to-transient rates.  It is the
// exact time reference of the world model's learned increment (Eq. 7 plug-in identity).
//
// Solver: BiCGSTAB with Jacobi preconditioning, the whole iteration inside ONE CTA (1024 threads): the spaces
// this is for (enumerable lattices, 1e3-1e6 states) fit one SM's work per iteration, every reduction has a
// fixed order (block tree), so the result is deterministic, and there is no host round trip per iteration.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include <vector>

#include "../../include/akmc.h"

namespace {

constexpr int kMT = 1024;

struct MfptParams {
    const int64_t* rp;
    const int32_t* col;
    const double* rate;
    int64_t n;
    double tol;
    int max_iter;
    double* x;          // tau
    double* r; double* rh; double* p; double* v; double* s; double* t; double* y; double* z; double* dinv;
    double* out;        // [0] relative residual, [1] iterations
};

// fixed-order block reduction of 1024 per-thread partials (deterministic)
__device__ double block_sum(double v, double* red)
{
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        double u = red[lane];
        for (int o = 16; o > 0; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
        if (lane == 0) red[32] = u;
    }
    __syncthreads();
    return red[32];
}

// y = A x with A = D - R (rows: diagonal = sum of all outgoing rates, off-diagonal = -rate to transient cols)
__device__ void spmv(const MfptParams& P, const double* x, double* yv)
{
    for (int64_t i = threadIdx.x; i < P.n; i += kMT) {
        double diag = 0.0, off = 0.0;
        for (int64_t e = P.rp[i]; e < P.rp[i + 1]; ++e) {
            const double g = P.rate[e];
            diag += g;
            const int32_t c = P.col[e];
            if (c >= 0) off = fma(g, x[c], off);
        }
        yv[i] = fma(diag, x[i], -off);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kMT) mfpt_bicgstab_kernel(const MfptParams P)
{
    __shared__ double red[33];
    const int tid = threadIdx.x;
    const int64_t n = P.n;
    // Jacobi preconditioner, x0 = D^-1 1, r = 1 - A x0
    for (int64_t i = tid; i < n; i += kMT) {
        double d = 0.0;
        for (int64_t e = P.rp[i]; e < P.rp[i + 1]; ++e) d += P.rate[e];
        P.dinv[i] = 1.0 / d;
        P.x[i] = P.dinv[i];
    }
    __syncthreads();
    spmv(P, P.x, P.t);
    double loc = 0.0;
    for (int64_t i = tid; i < n; i += kMT) {
        const double ri = 1.0 - P.t[i];
        P.r[i] = ri; P.rh[i] = ri; P.p[i] = 0.0; P.v[i] = 0.0;
        loc += ri * ri;
    }
    const double bnorm = sqrt((double)n);
    double rnorm = sqrt(block_sum(loc, red));
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    int it = 0;
    while (it < P.max_iter && rnorm > P.tol * bnorm) {
        ++it;
        loc = 0.0;
        for (int64_t i = tid; i < n; i += kMT) loc += P.rh[i] * P.r[i];
        const double rho1 = block_sum(loc, red);
        if (rho1 == 0.0) break;
        const double beta = (rho1 / rho) * (alpha / omega);
        rho = rho1;
        for (int64_t i = tid; i < n; i += kMT) {
            P.p[i] = P.r[i] + beta * (P.p[i] - omega * P.v[i]);
            P.y[i] = P.dinv[i] * P.p[i];
        }
        __syncthreads();
        spmv(P, P.y, P.v);
        loc = 0.0;
        for (int64_t i = tid; i < n; i += kMT) loc += P.rh[i] * P.v[i];
        const double rv = block_sum(loc, red);
        if (rv == 0.0) break;
        alpha = rho / rv;
        for (int64_t i = tid; i < n; i += kMT) {
            P.s[i] = P.r[i] - alpha * P.v[i];
            P.z[i] = P.dinv[i] * P.s[i];
        }
        __syncthreads();
        spmv(P, P.z, P.t);
        double ts = 0.0, tt = 0.0;
        for (int64_t i = tid; i < n; i += kMT) { ts += P.t[i] * P.s[i]; tt += P.t[i] * P.t[i]; }
        ts = block_sum(ts, red);
        tt = block_sum(tt, red);
        omega = tt > 0.0 ? ts / tt : 0.0;
        loc = 0.0;
        for (int64_t i = tid; i < n; i += kMT) {
            P.x[i] += alpha * P.y[i] + omega * P.z[i];
            const double ri = P.s[i] - omega * P.t[i];
            P.r[i] = ri;
            loc += ri * ri;
        }
        rnorm = sqrt(block_sum(loc, red));
        if (omega == 0.0) break;
    }
    // true residual of Eq. 5 with the final tau
    spmv(P, P.x, P.t);
    loc = 0.0;
    for (int64_t i = tid; i < n; i += kMT) { const double ri = 1.0 - P.t[i]; loc += ri * ri; }
    const double tr = sqrt(block_sum(loc, red));
    if (tid == 0) { P.out[0] = tr / bnorm; P.out[1] = (double)it; }
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
    if (e == cudaSuccess) e = cudaMalloc(&d_vec, ((size_t)10 * n + 2) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(d_rp, row_ptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(d_col, col, (size_t)nnz * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(d_rate, rate, (size_t)nnz * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        MfptParams P{};
        P.rp = d_rp; P.col = d_col; P.rate = d_rate; P.n = n; P.tol = tol; P.max_iter = max_iter;
        double* b = d_vec;
        P.x = b; P.r = b + n; P.rh = b + 2 * n; P.p = b + 3 * n; P.v = b + 4 * n; P.s = b + 5 * n; P.t = b + 6 * n;
        P.y = b + 7 * n; P.z = b + 8 * n; P.dinv = b + 9 * n; P.out = b + 10 * n;
        mfpt_bicgstab_kernel<<<1, kMT>>>(P);
        e = cudaGetLastError();
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
