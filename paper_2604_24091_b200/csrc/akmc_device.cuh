// akmc_device.cuh -- device primitives of the B200 AKMC path (sm_100a).
//
// Philox4x32-10 (reading A16, Salmon et al. SC'11), deterministic exp/log (A29), the
// geometry tables (window offsets P:561 / A3-A4, pair-KRA slot lists S:126-144) and the
// BKL tree (A17).  Every FP64 operation on the bit-exact path is an explicit IEEE intrinsic
// (__dadd_rn / __dmul_rn / __ddiv_rn / __fma_rn) so nvcc can neither contract nor reorder it;
// the operation order is the one DESIGN.md sec. 5 specifies.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace akmc {

constexpr int kSpecies = 7;
constexpr int kVac = 6;
constexpr int kFe = 0;
constexpr int kWin = 64;
constexpr int kHid = 256;
constexpr int kHops = 8;
constexpr int kPairTerms = 26;   // 7 + 6 (vacancy side) + 7 + 6 (target side)

// Geometry tables, passed to kernels by value (constant bank).
struct GeomTables {
    int8_t off[kWin][4];                 // hx, hy, hz (half-cell units), h^2
    int8_t pair_slot[kHops][kPairTerms]; // window slot of each counted neighbour
    int8_t pair_shell[kHops][kPairTerms];// 0 = 1NN, 1 = 2NN
    int8_t pair_sign[kHops][kPairTerms]; // +1 vacancy side, -1 target side
};

// Physical parameters (FP64), by value.
struct PhysParams {
    double Dp[2][kSpecies][kSpecies];    // Fe-referenced pair table (A.14)
    double E0[kSpecies];
    double kT;                           // kB * T (IEEE product, computed once on the host)
    double nu0;
    double inv_kT;                       // 1 / kT (FP32-equivalent mode only; FP64 mode divides, A29)
    const double* kT_vox;                // [n_voxels] kB * T_v (C4 per-voxel temperature; always set by init)
    const double* inv_kT_vox;            // [n_voxels] 1 / (kB * T_v) (FP32-equivalent evaluators only)
};

// Lattice frame of one voxel.  The voxel's L^3 owned cells are stored inside a halo of kHalo cells
// per face (storage (L + 2 kHalo)^3 cells x 2 basis, x fastest): the halo holds the periodic images
// (ghosts), so every 64-site window of an owned vacancy is a plain linear offset.
constexpr int kHalo = 2;                 // window reach: |h| <= 4 half-cells -> 2 cells
// Storage is bricked: 4x4x4 cells x 2 basis = 128 B = one L2 line per brick, bricks
// x-fastest; inside a brick the byte is ((z*4 + y)*4 + x)*2 + b.  A 64-site window touches ~8-12 lines.
struct Frame {
    int L[3];                            // owned cells
    int Ls[3];                           // storage cells = roundup4(L + 2*kHalo)
    int NB[3];                           // bricks per axis = Ls / 4
    int64_t sites;                       // storage sites (bytes) per voxel = 128 * NB0*NB1*NB2
    int wrap[3];                         // 1: axis periodic within this voxel (ghost images); 0: halo holds
                                         //    a neighbour rank's cells (multi-GPU spatial decomposition)
};

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// u_sel in [0,1) from words (0,1); u_t in (0,1] from words (2,3)  (A16, A18)
__device__ __forceinline__ void philox_uniforms(uint64_t seed, uint4 ctr, double& u_sel, double& u_t)
{
    const uint4 x = philox4x32_10(ctr, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const uint64_t a = ((uint64_t)x.x << 32) | x.y;
    const uint64_t b = ((uint64_t)x.z << 32) | x.w;
    u_sel = __dmul_rn((double)(a >> 11), 0x1.0p-53);
    u_t = __dmul_rn((double)((b >> 11) + 1ull), 0x1.0p-53);
}

// ------------------------------------------------------------------ det_exp / det_log (A29)
__device__ __forceinline__ double det_exp(double x)
{
    // Taylor coefficients 1/j!, j = 0..13, correctly rounded
    const double c13 = 0x1.6124613a86d09p-33, c12 = 0x1.1eed8eff8d898p-29, c11 = 0x1.ae64567f544e4p-26,
                 c10 = 0x1.27e4fb7789f5cp-22, c9 = 0x1.71de3a556c734p-19, c8 = 0x1.a01a01a01a01ap-16,
                 c7 = 0x1.a01a01a01a01ap-13, c6 = 0x1.6c16c16c16c17p-10, c5 = 0x1.1111111111111p-7,
                 c4 = 0x1.5555555555555p-5, c3 = 0x1.5555555555555p-3, c2 = 0x1.0p-1, c1 = 1.0, c0 = 1.0;
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const double inv_ln2 = 0x1.71547652b82fep+0;
    if (x < -700.0) x = -700.0;
    const double k = rint(__dmul_rn(x, inv_ln2));
    double r = __fma_rn(-k, ln2_hi, x);
    r = __fma_rn(-k, ln2_lo, r);
    double p = c13;
    p = __fma_rn(p, r, c12); p = __fma_rn(p, r, c11); p = __fma_rn(p, r, c10);
    p = __fma_rn(p, r, c9);  p = __fma_rn(p, r, c8);  p = __fma_rn(p, r, c7);
    p = __fma_rn(p, r, c6);  p = __fma_rn(p, r, c5);  p = __fma_rn(p, r, c4);
    p = __fma_rn(p, r, c3);  p = __fma_rn(p, r, c2);  p = __fma_rn(p, r, c1);
    p = __fma_rn(p, r, c0);
    // p * 2^k: for |k| <= 1000 (every caller's range) 2^k is a normal double and the product with p in [0.7, 1.5)
    // is exact and normal, so one multiply by the constructed power gives ldexp's bits
    const int ki = (int)k;
    if (ki >= -1000 && ki <= 1000) return __dmul_rn(p, __longlong_as_double((long long)(ki + 1023) << 52));
    return ldexp(p, ki);
}

__device__ __forceinline__ double det_log(double u)
{
    // odd series coefficients 1/(2j+1), j = 0..11
    const double d11 = 0x1.642c8590b2164p-5, d10 = 0x1.8618618618618p-5, d9 = 0x1.af286bca1af28p-5,
                 d8 = 0x1.e1e1e1e1e1e1ep-5, d7 = 0x1.1111111111111p-4, d6 = 0x1.3b13b13b13b14p-4,
                 d5 = 0x1.745d1745d1746p-4, d4 = 0x1.c71c71c71c71cp-4, d3 = 0x1.2492492492492p-3,
                 d2 = 0x1.999999999999ap-3, d1 = 0x1.5555555555555p-2, d0 = 1.0;
    const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
    const double sqrt_half = 0x1.6a09e667f3bcdp-1;
    int e;
    double m = frexp(u, &e);
    if (m < sqrt_half) { m = __dmul_rn(m, 2.0); e = e - 1; }
    const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
    const double z = __dmul_rn(s, s);
    double q = d11;
    q = __fma_rn(q, z, d10); q = __fma_rn(q, z, d9); q = __fma_rn(q, z, d8);
    q = __fma_rn(q, z, d7);  q = __fma_rn(q, z, d6); q = __fma_rn(q, z, d5);
    q = __fma_rn(q, z, d4);  q = __fma_rn(q, z, d3); q = __fma_rn(q, z, d2);
    q = __fma_rn(q, z, d1);  q = __fma_rn(q, z, d0);
    const double lm = __dmul_rn(2.0, __dmul_rn(s, q));
    const double de = (double)e;
    return __fma_rn(de, ln2_hi, __fma_rn(de, ln2_lo, lm));
}

// kT of the voxel a vacancy lives in (SURVEY 8(d) C4 variant: per-voxel T); vox < 0 (a bare
// window, akmc_eval_windows) -> the configured T
__device__ __forceinline__ double kT_of(const PhysParams& P, int vox)
{
    return vox >= 0 ? __ldg(P.kT_vox + vox) : P.kT;
}

// FP32-equivalent evaluators (tensor-core paths; the 1e-5 bar, not bit-exact with the oracle): the exponent is
// E * (1 / kT_v) -- one multiply instead of an FP64 division (relative change of the rate ~|E/kT| ulp ~ 1e-15)
__device__ __forceinline__ double arrhenius_tc(double E, const PhysParams& P, int vox)
{
    const double ik = vox >= 0 ? __ldg(P.inv_kT_vox + vox) : P.inv_kT;
    return __dmul_rn(P.nu0, det_exp(-__dmul_rn(E, ik)));
}

// Gamma = nu0 * det_exp(-(E / kT_v)), masked -> exactly 0 (Eq. 1; Eq. 8)
__device__ __forceinline__ double arrhenius(double E, const PhysParams& P, int vox)
{
    return __dmul_rn(P.nu0, det_exp(-__ddiv_rn(E, kT_of(P, vox))));
}

// ------------------------------------------------------------------ lattice addressing
// vacancy position: x = voxel, y/z/w = OWNED half-cell coordinates px, py, pz in [0, 2L)
__device__ __forceinline__ int wrap2(int p, int twoL) { return p < 0 ? p + twoL : (p >= twoL ? p - twoL : p); }

// storage site of owned half-cell coordinates (p may reach kHalo cells outside [0, 2L))
__device__ __forceinline__ int64_t site_of(const Frame& F, int vox, int px, int py, int pz)
{
    const int cx = (px >> 1) + kHalo, cy = (py >> 1) + kHalo, cz = (pz >> 1) + kHalo;
    // brick index < 2^25 for any allowed block (32-bit math); only the byte offset needs 64 bits
    const uint32_t brick = (uint32_t)(cx >> 2) + (uint32_t)F.NB[0] * ((uint32_t)(cy >> 2) + (uint32_t)F.NB[1] * (uint32_t)(cz >> 2));
    const int inb = ((((cz & 3) << 2) | (cy & 3)) << 3) | ((cx & 3) << 1) | (px & 1);
    return (int64_t)vox * F.sites + ((int64_t)brick << 7) + inb;
}

// window site of an owned vacancy: no wrap needed, the halo holds the periodic images
__device__ __forceinline__ int64_t neighbour_site(const Frame& F, const int4& v, int dx, int dy, int dz)
{
    return site_of(F, v.x, v.y + dx, v.z + dy, v.w + dz);
}

// write an owned site and all its ghost images in the halo (periodic voxel)
__device__ __forceinline__ void write_site(uint8_t* species, const Frame& F, int vox, int px, int py, int pz, uint8_t val)
{
    int ix[2], iy[2], iz[2];
    int nx = 1, ny = 1, nz = 1;
    ix[0] = px; iy[0] = py; iz[0] = pz;
    const int cx = px >> 1, cy = py >> 1, cz = pz >> 1;
    if (F.wrap[0]) { if (cx < kHalo) ix[nx++] = px + 2 * F.L[0]; else if (cx >= F.L[0] - kHalo) ix[nx++] = px - 2 * F.L[0]; }
    if (F.wrap[1]) { if (cy < kHalo) iy[ny++] = py + 2 * F.L[1]; else if (cy >= F.L[1] - kHalo) iy[ny++] = py - 2 * F.L[1]; }
    if (F.wrap[2]) { if (cz < kHalo) iz[nz++] = pz + 2 * F.L[2]; else if (cz >= F.L[2] - kHalo) iz[nz++] = pz - 2 * F.L[2]; }
    for (int a = 0; a < nx; ++a)
        for (int b = 0; b < ny; ++b)
            for (int c = 0; c < nz; ++c) species[site_of(F, vox, ix[a], iy[b], iz[c])] = val;
}

// ------------------------------------------------------------------ pair KRA barrier
// E_k = max(0, E0[X] + 0.5 * sum_{s,y} dc[s][y] * Dp[s][X][y]); dc from the window (A.1).
// returns 1 if clamped (pre-clamp < 0)
__device__ __forceinline__ int pair_barrier(const uint8_t* w, int k, const GeomTables& G, const PhysParams& P, double& E)
{
    const int X = w[k];
    int dc[2][kSpecies];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int y = 0; y < kSpecies; ++y) dc[s][y] = 0;
#pragma unroll
    for (int t = 0; t < kPairTerms; ++t) {
        const int sl = G.pair_slot[k][t];
        const int sh = G.pair_shell[k][t];
        dc[sh][w[sl]] += G.pair_sign[k][t];
    }
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int y = 0; y < kSpecies; ++y) acc = __fma_rn((double)dc[s][y], P.Dp[s][X][y], acc);
    const double e = __dadd_rn(P.E0[X], __dmul_rn(0.5, acc));
    if (e < 0.0) { E = 0.0; return 1; }
    E = (e > 0.0) ? e : 0.0;
    return 0;
}

} // namespace akmc
