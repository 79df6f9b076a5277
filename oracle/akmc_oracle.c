/*
 * akmc_oracle.c -- plain, slow, single-threaded FP64 CPU ORACLE for the AKMC
 * vacancy-hop step of AtomWorld (arXiv 2604.24091).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2604_24091_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * What it computes (citations: P:NNN = /root/reference/PAPER.md line,
 * S:NNN = SPEC.md line; readings A1..A30 are listed in DESIGN.md sec. 3):
 *   - bcc lattice, canonical site index 2*(x + Lx*(y + Ly*z)) + b  (A1)
 *   - 64-site window of shells 1..6 within 6.0 A, a0 = 2.866 A (A3, A4)
 *   - pair KRA barrier E = max(0, E0[X] + dE/2) with the broken-bond pair model
 *     on shells 1-2 (A10-A12), computed from the lattice itself
 *   - FP64 barrier MLP 448-256-256-8 ReLU on the one-hot window (A8)
 *   - Arrhenius rate nu0*exp(-E/kT) (Eq. 8)
 *   - residence-time (BKL) selection = Eq. 2 with log-rate logits (P:294-298,
 *     S:195-203), Philox4x32-10 counters (A16), pairwise tree (A17)
 *   - windowed synchronous sublattice sweeps (reading A19)
 *   - Cu cluster statistics
 * Every floating-point step is written in the order the DESIGN.md spec fixes;
 * this file is compiled with -ffp-contract=off so only explicit fma() fuses.
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, brute force, paper and
 * SPEC worked examples, Random123 KATs).  No function here is "parity
 * unpinned" except where stated in its comment.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef ORC_MUTANT
#define ORC_MUTANT 0   /* test-only fault injection (tests/test_oracle_selection.py); 0 in every real build */
#endif

#define NSPEC 7   /* Fe0 Cu1 Ni2 Mn3 Si4 P5 V6 (A6) */
#define VAC 6
#define FE 0
#define NWIN 64
#define NHID 256

/* ------------------------------------------------------------------ */
/* configuration (the oracle's own struct; not shared with the GPU)    */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t cells[3];     /* Lx, Ly, Lz bcc cells per voxel */
    int32_t n_voxels;     /* independent periodic voxels */
    double  T;            /* K */
    double  nu0;          /* 1/s */
    double  kB;           /* eV/K */
    int32_t model;        /* 0 pair KRA, 1 MLP */
    int32_t domain[3];    /* sublattice domain edge in cells, 0 => serial BKL */
    double  window_s;     /* Delta_win per phase */
    uint64_t seed;        /* Philox key */
    int32_t strict;       /* 1: recompute active sets by full scan (slow, checks A20) */
    const double* voxel_T;/* [n_voxels] K per voxel or NULL (= T everywhere): the C4 variant with
                             per-voxel temperature ("temperatures ... vary") */
} orc_cfg;

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. SC'11; Random123 constants; A16)        */
/* ------------------------------------------------------------------ */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw_uniforms(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                          double* u_sel, double* u_t)
{
    uint32_t ctr[4] = {a, b, c, d};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    orc_philox(ctr, key, x);
    uint64_t w01 = ((uint64_t)x[0] << 32) | x[1];
    uint64_t w23 = ((uint64_t)x[2] << 32) | x[3];
    *u_sel = (double)(w01 >> 11) * 0x1.0p-53;         /* [0,1)  */
    *u_t = (double)((w23 >> 11) + 1) * 0x1.0p-53;      /* (0,1]  (A18) */
}

/* ------------------------------------------------------------------ */
/* deterministic exp / log (A29): fixed op order, explicit fma          */
/* ------------------------------------------------------------------ */
static const double EXP_C[14] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};
static const double LOG_C[12] = {
    0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
static const double LN2_HI = 0x1.62e42fee00000p-1;
static const double LN2_LO = 0x1.a39ef35793c76p-33;
static const double INV_LN2 = 0x1.71547652b82fep+0;
static const double SQRT_HALF = 0x1.6a09e667f3bcdp-1;

double orc_det_exp(double x)
{
    if (x < -700.0) x = -700.0;
    double k = nearbyint(x * INV_LN2);
    double r = fma(-k, LN2_HI, x);
    r = fma(-k, LN2_LO, r);
    double p = EXP_C[13];
    for (int j = 12; j >= 0; --j) p = fma(p, r, EXP_C[j]);
    return ldexp(p, (int)k);
}

double orc_det_log(double u)
{
    int e;
    double m = frexp(u, &e);
    if (m < SQRT_HALF) { m = m * 2.0; e = e - 1; }
    double s = (m - 1.0) / (m + 1.0);
    double z = s * s;
    double q = LOG_C[11];
    for (int j = 10; j >= 0; --j) q = fma(q, z, LOG_C[j]);
    double lm = 2.0 * (s * q);
    double de = (double)e;
    return fma(de, LN2_HI, fma(de, LN2_LO, lm));
}

/* array forms of the two (test convenience: one call instead of n ctypes calls) */
void orc_det_exp_n(const double* x, int64_t n, double* y) { for (int64_t i = 0; i < n; ++i) y[i] = orc_det_exp(x[i]); }
void orc_det_log_n(const double* x, int64_t n, double* y) { for (int64_t i = 0; i < n; ++i) y[i] = orc_det_log(x[i]); }

/* ------------------------------------------------------------------ */
/* geometry                                                             */
/* ------------------------------------------------------------------ */
/* half-cell offsets of the 64-site window: all bcc vectors (all-even or all-odd
 * half-cell components) with |r| <= 6.0 A at a0 = 2.866 A, sorted by
 * (|h|^2, hx, hy, hz) (A4).  Slots 0..7 are the 1NN, slot k = 4[hx>0]+2[hy>0]+[hz>0]. */
static int g_win[NWIN][3];
static int g_win_h2[NWIN];
static int g_win_ready = 0;

static int cmp_off(const void* a, const void* b)
{
    const int* p = (const int*)a;
    const int* q = (const int*)b;
    for (int i = 0; i < 4; ++i) {
        if (p[i] != q[i]) return p[i] < q[i] ? -1 : 1;
    }
    return 0;
}

static void build_window(void)
{
    if (g_win_ready) return;
    int tmp[200][4];
    int n = 0;
    const double a0 = 2.866, rc = 6.0;
    for (int hx = -6; hx <= 6; ++hx)
        for (int hy = -6; hy <= 6; ++hy)
            for (int hz = -6; hz <= 6; ++hz) {
                int ax = hx & 1, ay = hy & 1, az = hz & 1;
                if (!(ax == ay && ay == az)) continue;       /* bcc: same parity */
                if (hx == 0 && hy == 0 && hz == 0) continue;
                int h2 = hx * hx + hy * hy + hz * hz;
                double r = sqrt((double)h2) * a0 / 2.0;
                if (r <= rc) {
                    tmp[n][0] = h2; tmp[n][1] = hx; tmp[n][2] = hy; tmp[n][3] = hz;
                    ++n;
                }
            }
    qsort(tmp, (size_t)n, sizeof(tmp[0]), cmp_off);
    /* n must be 64 (pinned by tests) */
    for (int i = 0; i < n && i < NWIN; ++i) {
        g_win_h2[i] = tmp[i][0];
        g_win[i][0] = tmp[i][1]; g_win[i][1] = tmp[i][2]; g_win[i][2] = tmp[i][3];
    }
    g_win_ready = (n == NWIN) ? 1 : -1;
}

int orc_window_offsets(int32_t* out /* [64][4] = hx,hy,hz,h2 */)
{
    build_window();
    if (g_win_ready != 1) return -1;
    for (int i = 0; i < NWIN; ++i) {
        out[4 * i + 0] = g_win[i][0]; out[4 * i + 1] = g_win[i][1];
        out[4 * i + 2] = g_win[i][2]; out[4 * i + 3] = g_win_h2[i];
    }
    return NWIN;
}

typedef struct { int64_t sites_per_voxel; int L[3]; } geom;

static geom mk_geom(const orc_cfg* c)
{
    geom g;
    g.L[0] = c->cells[0]; g.L[1] = c->cells[1]; g.L[2] = c->cells[2];
    g.sites_per_voxel = 2LL * g.L[0] * g.L[1] * g.L[2];
    return g;
}

/* global site index -> voxel and half-cell position p = 2*cell + basis */
static void site_pos(const geom* g, int64_t site, int64_t* vox, int p[3])
{
    int64_t v = site / g->sites_per_voxel;
    int64_t i = site - v * g->sites_per_voxel;
    int b = (int)(i & 1);
    int64_t cell = i >> 1;
    int x = (int)(cell % g->L[0]);
    int64_t t = cell / g->L[0];
    int y = (int)(t % g->L[1]);
    int z = (int)(t / g->L[1]);
    *vox = v;
    p[0] = 2 * x + b; p[1] = 2 * y + b; p[2] = 2 * z + b;
}

static int64_t pos_site(const geom* g, int64_t vox, const int p[3])
{
    int q[3];
    for (int a = 0; a < 3; ++a) {
        int m = 2 * g->L[a];
        q[a] = ((p[a] % m) + m) % m;   /* periodic wrap */
    }
    int b = q[0] & 1;
    int64_t cell = (int64_t)(q[0] >> 1) + (int64_t)g->L[0] * ((int64_t)(q[1] >> 1) + (int64_t)g->L[1] * (int64_t)(q[2] >> 1));
    return vox * g->sites_per_voxel + 2 * cell + b;
}

/* sites of shell s (1 or 2) around a site: 1NN offsets (+-1,+-1,+-1), 2NN (+-2,0,0)... */
static const int NN1[8][3] = {{-1,-1,-1},{-1,-1,1},{-1,1,-1},{-1,1,1},{1,-1,-1},{1,-1,1},{1,1,-1},{1,1,1}};
static const int NN2[6][3] = {{-2,0,0},{2,0,0},{0,-2,0},{0,2,0},{0,0,-2},{0,0,2}};

/* ------------------------------------------------------------------ */
/* energetics                                               */
/* ------------------------------------------------------------------ */
/* eps layout: eps[s][a][b], s = 0 (1NN) / 1 (2NN), 7x7 each, eV.          */
#define EPS(e, s, a, b) ((e)[((s) * NSPEC + (a)) * NSPEC + (b)])

/* total pair energy of one voxel: every unordered 1NN and 2NN bond once */
double orc_system_energy(const orc_cfg* c, const uint8_t* species, int64_t vox, const double* eps)
{
    geom g = mk_geom(c);
    double E = 0.0;
    for (int64_t i = 0; i < g.sites_per_voxel; ++i) {
        int64_t site = vox * g.sites_per_voxel + i;
        int64_t vv; int p[3];
        site_pos(&g, site, &vv, p);
        int a = species[site];
        for (int j = 0; j < 8; ++j) {
            int q[3] = {p[0] + NN1[j][0], p[1] + NN1[j][1], p[2] + NN1[j][2]};
            int64_t t = pos_site(&g, vox, q);
            if (t > site) E += EPS(eps, 0, a, species[t]);
        }
        for (int j = 0; j < 6; ++j) {
            int q[3] = {p[0] + NN2[j][0], p[1] + NN2[j][1], p[2] + NN2[j][2]};
            int64_t t = pos_site(&g, vox, q);
            if (t > site) E += EPS(eps, 1, a, species[t]);
        }
    }
    return E;
}

/* integer count differences dc[s][y] = #{shell-s neighbours of v, != n, species y}
 *                                     - #{shell-s neighbours of n, != v, species y}
 * taken straight from the lattice. */
static void count_dc(const geom* g, const uint8_t* sp, int64_t vox, const int pv[3], const int pn[3],
                     int64_t vsite, int64_t nsite, int dc[2][NSPEC])
{
    memset(dc, 0, sizeof(int) * 2 * NSPEC);
    for (int j = 0; j < 8; ++j) {
        int q[3] = {pv[0] + NN1[j][0], pv[1] + NN1[j][1], pv[2] + NN1[j][2]};
        int64_t t = pos_site(g, vox, q);
        if (t != nsite) dc[0][sp[t]] += 1;
        int r[3] = {pn[0] + NN1[j][0], pn[1] + NN1[j][1], pn[2] + NN1[j][2]};
        int64_t u = pos_site(g, vox, r);
        if (u != vsite) dc[0][sp[u]] -= 1;
    }
    for (int j = 0; j < 6; ++j) {
        int q[3] = {pv[0] + NN2[j][0], pv[1] + NN2[j][1], pv[2] + NN2[j][2]};
        int64_t t = pos_site(g, vox, q);
        if (t != nsite) dc[1][sp[t]] += 1;
        int r[3] = {pn[0] + NN2[j][0], pn[1] + NN2[j][1], pn[2] + NN2[j][2]};
        int64_t u = pos_site(g, vox, r);
        if (u != vsite) dc[1][sp[u]] -= 1;
    }
}

/* dE of swapping the vacancy at vsite with the atom in 1NN direction k, using the
 * plain D[s][X][y] = eps[s][X][y] - eps[s][V][y]; used by the pins. */
double orc_delta_energy(const orc_cfg* c, const uint8_t* sp, int64_t vsite, int k, const double* eps)
{
    geom g = mk_geom(c);
    int64_t vox; int pv[3];
    site_pos(&g, vsite, &vox, pv);
    build_window();
    int pn[3] = {pv[0] + g_win[k][0], pv[1] + g_win[k][1], pv[2] + g_win[k][2]};
    int64_t nsite = pos_site(&g, vox, pn);
    int X = sp[nsite];
    int dc[2][NSPEC];
    count_dc(&g, sp, vox, pv, pn, vsite, nsite, dc);
    double acc = 0.0;
    for (int s = 0; s < 2; ++s)
        for (int y = 0; y < NSPEC; ++y)
            acc = fma((double)dc[s][y], EPS(eps, s, X, y) - EPS(eps, s, VAC, y), acc);
    return acc;
}

/* Fe-referenced table Dp[s][X][y] = (eps[s][X][y] - eps[s][V][y]) - (eps[s][X][Fe] - eps[s][V][Fe])
 * (A.14: exact because sum_y dc[s][y] = 0 in every shell). */
static void build_dp(const double* eps, double* Dp)
{
    for (int s = 0; s < 2; ++s)
        for (int X = 0; X < NSPEC; ++X)
            for (int y = 0; y < NSPEC; ++y) {
                double d = EPS(eps, s, X, y) - EPS(eps, s, VAC, y);
                double dfe = EPS(eps, s, X, FE) - EPS(eps, s, VAC, FE);
                Dp[(s * NSPEC + X) * NSPEC + y] = d - dfe;
            }
}

/* window sigma[64] around vsite */
static void window_of(const geom* g, const uint8_t* sp, int64_t vsite, uint8_t sigma[NWIN])
{
    int64_t vox; int pv[3];
    site_pos(g, vsite, &vox, pv);
    for (int j = 0; j < NWIN; ++j) {
        int q[3] = {pv[0] + g_win[j][0], pv[1] + g_win[j][1], pv[2] + g_win[j][2]};
        sigma[j] = sp[pos_site(g, vox, q)];
    }
}

int orc_window(const orc_cfg* c, const uint8_t* sp, int64_t vsite, uint8_t* sigma)
{
    build_window();
    geom g = mk_geom(c);
    window_of(&g, sp, vsite, sigma);
    return 0;
}

/* FP64 MLP 448-256-256-8 (A8): dense loop over all 448 one-hot features
 * in ascending feature order f = 7*slot + species, acc = fma(x_f, W[f][j], acc). */
static void mlp_forward(const uint8_t sigma[NWIN], const double* mlp, double out[8]);

void orc_mlp_fp64(const uint8_t sigma[NWIN], const double* mlp, double E[8])
{
    double out[8];
    mlp_forward(sigma, mlp, out);
    for (int k = 0; k < 8; ++k) E[k] = out[k] > 0.0 ? out[k] : 0.0;    /* barrier reading: clamp at 0 (A8) */
}

/* raw network outputs (no clamp): the barrier reading clamps them, the world-model reading uses them as the
 * policy logits z_{i,k} of Eq. 1 */
static void mlp_forward(const uint8_t sigma[NWIN], const double* mlp, double out[8])
{
    const double* W1 = mlp;
    const double* b1 = W1 + 448 * NHID;
    const double* W2 = b1 + NHID;
    const double* b2 = W2 + NHID * NHID;
    const double* W3 = b2 + NHID;
    const double* b3 = W3 + NHID * 8;
    double h1[NHID], h2[NHID];
    for (int j = 0; j < NHID; ++j) {
        double acc = b1[j];
        for (int f = 0; f < 448; ++f) {
            double x = (sigma[f / 7] == (uint8_t)(f % 7)) ? 1.0 : 0.0;
            acc = fma(x, W1[(size_t)f * NHID + j], acc);
        }
        h1[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < NHID; ++j) {
        double acc = b2[j];
        for (int i = 0; i < NHID; ++i) acc = fma(h1[i], W2[(size_t)i * NHID + j], acc);
        h2[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int k = 0; k < 8; ++k) {
        double acc = b3[k];
        for (int i = 0; i < NHID; ++i) acc = fma(h2[i], W3[(size_t)i * 8 + k], acc);
        out[k] = acc;
    }
}

/* barriers and rates of the 8 hops of one vacancy; returns the number of clamps */
static int vac_rates(const orc_cfg* c, const geom* g, const uint8_t* sp, int64_t vsite,
                     const double* Dp, const double* E0, const double* mlp,
                     double E[8], double G[8])
{
    int64_t vox; int pv[3];
    site_pos(g, vsite, &vox, pv);
    int clamps = 0;
    uint8_t sigma[NWIN];
    if (c->model == 1) {
        window_of(g, sp, vsite, sigma);
        orc_mlp_fp64(sigma, mlp, E);
    }
    double kT = c->kB * (c->voxel_T ? c->voxel_T[vox] : c->T);   /* the vacancy's voxel's T */
    for (int k = 0; k < 8; ++k) {
        int pn[3] = {pv[0] + g_win[k][0], pv[1] + g_win[k][1], pv[2] + g_win[k][2]};
        int64_t nsite = pos_site(g, vox, pn);
        int X = sp[nsite];
        if (c->model == 0) {
            if (X == VAC) {
                E[k] = 0.0;
            } else {
                int dc[2][NSPEC];
                count_dc(g, sp, vox, pv, pn, vsite, nsite, dc);
                double acc = 0.0;
                for (int s = 0; s < 2; ++s)
                    for (int y = 0; y < NSPEC; ++y)
                        acc = fma((double)dc[s][y], Dp[(s * NSPEC + X) * NSPEC + y], acc);
                double e = E0[X] + 0.5 * acc;
                if (e < 0.0) { clamps += 1; e = 0.0; } else if (!(e > 0.0)) { e = 0.0; }
                E[k] = e;
            }
        }
        if (X == VAC) {
            G[k] = 0.0;                                    /* mask m_k = 0 (A14) */
        } else {
            G[k] = c->nu0 * orc_det_exp(-(E[k] / kT));     /* Eq. 8 */
        }
    }
    return clamps;
}

int orc_barriers(const orc_cfg* c, const uint8_t* sp, int64_t vsite, const double* eps,
                 const double* E0, const double* mlp, double* E, double* G)
{
    build_window();
    if (g_win_ready != 1) return -1;
    geom g = mk_geom(c);
    double Dp[2 * NSPEC * NSPEC];
    if (eps) build_dp(eps, Dp);
    return vac_rates(c, &g, sp, vsite, Dp, E0, mlp, E, G);
}

/* ------------------------------------------------------------------ */
/* canonical pairwise tree + descent (A17)                              */
/* ------------------------------------------------------------------ */
typedef struct { double* lv; int P; int levels; } tree_t;

/* leaves R[0..n-1] padded with 0 to P = 2^ceil(log2 n); node = left + right */
static double tree_build(const double* R, int n, double* buf, int* P_out, int* levels_out)
{
    int P = 1, levels = 0;
    while (P < n) { P <<= 1; ++levels; }
#if ORC_MUTANT == 3   /* test-only mutant: the padded tree drops the last real leaf */
    for (int i = 0; i < P; ++i) buf[i] = (i < n - 1) ? R[i] : 0.0;
#else
    for (int i = 0; i < P; ++i) buf[i] = (i < n) ? R[i] : 0.0;
#endif
    int off = 0, width = P;
    while (width > 1) {
        for (int i = 0; i < width / 2; ++i) buf[off + width + i] = buf[off + 2 * i] + buf[off + 2 * i + 1];
        off += width;
        width /= 2;
    }
    *P_out = P; *levels_out = levels;
    return buf[off];
}

/* descend with r: at node (L,R) go left if r < L, else r -= L and go right.
 * guard: a reached leaf with R == 0 is replaced by the last leaf with R > 0. */
static int tree_descend(const double* buf, const double* R, int n, int P, double* r_io)
{
    /* level offsets: level 0 (leaves) at 0, width P; level l at sum_{j<l} P>>j */
    int nlev = 0; { int w = P; while (w > 1) { w >>= 1; ++nlev; } }
    int offs[64];
    int off = 0, w = P;
    for (int l = 0; l <= nlev; ++l) { offs[l] = off; off += w; w >>= 1; }
    double r = *r_io;
    int idx = 0;
    for (int l = nlev; l >= 1; --l) {
        double left = buf[offs[l - 1] + 2 * idx];
#if ORC_MUTANT == 1   /* test-only mutant: right turn keeps r (no subtraction of the left mass) */
        if (r < left) idx = 2 * idx; else idx = 2 * idx + 1;
#elif ORC_MUTANT == 2 /* test-only mutant: wrong child offset (children swapped) */
        if (r < left) { idx = 2 * idx + 1; } else { r = r - left; idx = 2 * idx; }
#else
        if (r < left) {
            idx = 2 * idx;
        } else {
            r = r - left;
            idx = 2 * idx + 1;
        }
#endif
    }
    if (idx >= n || !(R[idx] > 0.0)) {
        int last = -1;
        for (int i = 0; i < n; ++i) if (R[i] > 0.0) last = i;
        idx = last;
    }
    *r_io = r;
    return idx;
}

/* within vacancy: first k with r < cumsum_k (sequential), guard: last k with G > 0 */
static int pick_hop(const double G[8], double r)
{
    double cs = 0.0;
    for (int k = 0; k < 8; ++k) {
        cs = cs + G[k];
        if (r < cs) return k;
    }
    int last = -1;
    for (int k = 0; k < 8; ++k) if (G[k] > 0.0) last = k;
    return last;
}

/* One residence-time selection over n competing vacancies (Eq. 2 with log-rate logits, P:294-298;
 * S:195-198): R_i = sequential sum of the 8 hop rates G[i][0..7] (A17); Gamma_tot = canonical pairwise tree
 * over R_0..R_{n-1}; r = u_sel * Gamma_tot; descend to the vacancy, then pick_hop inside it.  This is exactly
 * the code path of run_serial / run_sublattice (they call tree_build / tree_descend / pick_hop in this order).
 * Returns Gamma_tot; *i_out = *k_out = -1 when Gamma_tot == 0 (terminal). */
double orc_bkl_select_u(const double* G, int n, double u_sel, int* i_out, int* k_out)
{
    double* R = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)(n + 2));
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k < 8; ++k) s = s + G[8 * i + k];
        R[i] = s;
    }
    int P = 1, lev = 0;
    double tot = (n > 0) ? tree_build(R, n, buf, &P, &lev) : 0.0;
    *i_out = -1; *k_out = -1;
    if (tot > 0.0) {
        double r = u_sel * tot;
        int a = tree_descend(buf, R, n, P, &r);
        *i_out = a;
        *k_out = pick_hop(&G[8 * a], r);
    }
    free(R); free(buf);
    return tot;
}

/* the serial-mode uniforms of one event (A16/A18): Philox4x32-10(key = seed; ctr = (c0, c1, c2, c3)) */
void orc_draw_uniforms(uint64_t seed, const uint32_t ctr[4], double* u_sel, double* u_t)
{
    draw_uniforms(seed, ctr[0], ctr[1], ctr[2], ctr[3], u_sel, u_t);
}

/* ------------------------------------------------------------------ */
/* runs                                                                 */
/* ------------------------------------------------------------------ */
enum { ORC_OK = 0, ORC_INVALID = 2, ORC_TERMINAL = 3 };

typedef struct {
    int64_t events, hop_evals, terminal_voxels, clamps;
} orc_ctr;

static void apply_hop(const geom* g, uint8_t* sp, int64_t* vac, int i, int k)
{
    int64_t vsite = vac[i];
    int64_t vox; int pv[3];
    site_pos(g, vsite, &vox, pv);
    int pn[3] = {pv[0] + g_win[k][0], pv[1] + g_win[k][1], pv[2] + g_win[k][2]};
    int64_t nsite = pos_site(g, vox, pn);
    uint8_t t = sp[vsite];
    sp[vsite] = sp[nsite];   /* swap */
    sp[nsite] = t;
    vac[i] = nsite;
}

/* serial BKL, one competing set per voxel (P:294-298 with A15).
 * Each voxel runs n events (or until Gamma_tot == 0 -> terminal).  With a horizon (t_end finite; the
 * voxel-ensemble mode of P:453-455, every voxel advanced to a common physical time) a voxel also stops
 * at the first draw whose event time clock + dt exceeds t_end; that draw is discarded and its counter
 * is not consumed, so horizons split a run without changing the trajectory. */
static int run_serial(const orc_cfg* c, uint8_t* sp, int64_t* vac, int64_t nvac, double* clock,
                      int64_t* nev, const double* Dp, const double* E0, const double* mlp,
                      int64_t n, double t_end, orc_ctr* ctr)
{
    geom g = mk_geom(c);
    int* members = (int*)malloc(sizeof(int) * (size_t)(nvac + 1));
    double* R = (double*)malloc(sizeof(double) * (size_t)(nvac + 1));
    double* G = (double*)malloc(sizeof(double) * 8 * (size_t)(nvac + 1));
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)(nvac + 2));
    int rc = ORC_OK;
    for (int64_t v = 0; v < c->n_voxels; ++v) {
        int m = 0;
        for (int64_t i = 0; i < nvac; ++i)
            if (vac[i] / g.sites_per_voxel == v) members[m++] = (int)i;
        for (int64_t e = 0; e < n; ++e) {
            for (int a = 0; a < m; ++a) {
                double E[8];
                ctr->clamps += vac_rates(c, &g, sp, vac[members[a]], Dp, E0, mlp, E, &G[8 * a]);
                double s = 0.0;
                for (int k = 0; k < 8; ++k) s = s + G[8 * a + k];
                R[a] = s;
            }
            ctr->hop_evals += 8LL * m;
            int P = 1, lev = 0;
            double tot = (m > 0) ? tree_build(R, m, buf, &P, &lev) : 0.0;
            if (!(tot > 0.0)) {      /* no feasible event */
                ctr->terminal_voxels += 1;
                rc = ORC_TERMINAL;
                break;
            }
            double u_sel, u_t;
            draw_uniforms(c->seed, (uint32_t)nev[v], (uint32_t)((uint64_t)nev[v] >> 32), (uint32_t)v, 0u,
                          &u_sel, &u_t);
            double dt = (-orc_det_log(u_t)) / tot;
            if (clock[v] + dt > t_end) break;   /* horizon: the event would happen after t_end */
            double r = u_sel * tot;
            int a = tree_descend(buf, R, m, P, &r);
            int k = pick_hop(&G[8 * a], r);
            apply_hop(&g, sp, vac, members[a], k);
            clock[v] = clock[v] + dt;
            nev[v] += 1;
            ctr->events += 1;
        }
    }
    free(members); free(R); free(G); free(buf);
    return rc;
}

/* sublattice bookkeeping: domain id and sector of the vacancy's current cell */
static void dom_sector(const orc_cfg* c, const geom* g, int64_t site, int64_t* dom, int* sec)
{
    int64_t vox; int p[3];
    site_pos(g, site, &vox, p);
    int nd[3], dcoord[3], o[3];
    for (int a = 0; a < 3; ++a) {
        int D = c->domain[a];
        int cell = p[a] >> 1;
        nd[a] = g->L[a] / D;
        dcoord[a] = cell / D;
        o[a] = (cell % D) >= D / 2 ? 1 : 0;
    }
    int64_t per_vox = (int64_t)nd[0] * nd[1] * nd[2];
    *dom = vox * per_vox + dcoord[0] + (int64_t)nd[0] * (dcoord[1] + (int64_t)nd[1] * dcoord[2]);
    *sec = o[0] | (o[1] << 1) | (o[2] << 2);
}

typedef struct { int64_t dom; int64_t slot; } dkey;
static int cmp_dkey(const void* a, const void* b)
{
    const dkey* p = (const dkey*)a;
    const dkey* q = (const dkey*)b;
    if (p->dom != q->dom) return p->dom < q->dom ? -1 : 1;
    if (p->slot != q->slot) return p->slot < q->slot ? -1 : 1;
    return 0;
}

void orc_sector_perm(uint64_t seed, int64_t sweep, int perm[8])
{
    uint32_t y[8];
    for (int j = 0; j < 2; ++j) {
        uint32_t ctr[4] = {(uint32_t)j, 0xFFFFFFFFu, (uint32_t)sweep, (uint32_t)((uint64_t)sweep >> 32)};
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        orc_philox(ctr, key, &y[4 * j]);
    }
    for (int i = 0; i < 8; ++i) perm[i] = i;
    for (int i = 7; i >= 1; --i) {
        int j = (int)(y[i] % (uint32_t)(i + 1));
        int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
}

/* windowed synchronous sublattice (reading A19) */
static int run_sublattice(const orc_cfg* c, uint8_t* sp, int64_t* vac, int64_t nvac, double* clock,
                          int64_t* sweep_io, const double* Dp, const double* E0, const double* mlp,
                          int64_t n, orc_ctr* ctr)
{
    geom g = mk_geom(c);
    dkey* keys = (dkey*)malloc(sizeof(dkey) * (size_t)(nvac + 1));
    int* A = (int*)malloc(sizeof(int) * (size_t)(nvac + 1));
    double* R = (double*)malloc(sizeof(double) * (size_t)(nvac + 1));
    double* G = (double*)malloc(sizeof(double) * 8 * (size_t)(nvac + 1));
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)(nvac + 2));
    for (int64_t sw = 0; sw < n; ++sw) {
        int64_t s = *sweep_io;
        int perm[8];
        orc_sector_perm(c->seed, s, perm);
        for (int q = 0; q < 8; ++q) {
            int64_t p = 8 * s + q;
            int csec = perm[q];
            /* active vacancies of this phase, grouped by domain, slot order */
            int64_t na = 0;
            for (int64_t i = 0; i < nvac; ++i) {
                int64_t d; int sc;
                dom_sector(c, &g, vac[i], &d, &sc);
                if (sc == csec) { keys[na].dom = d; keys[na].slot = i; ++na; }
            }
            qsort(keys, (size_t)na, sizeof(dkey), cmp_dkey);
            int64_t a0 = 0;
            while (a0 < na) {
                int64_t a1 = a0;
                while (a1 < na && keys[a1].dom == keys[a0].dom) ++a1;
                int64_t d = keys[a0].dom;
                double t = 0.0;
                uint32_t it = 0;
                for (;;) {
                    int m = 0;
                    if (c->strict) {
                        for (int64_t i = 0; i < nvac; ++i) {
                            int64_t dd; int sc;
                            dom_sector(c, &g, vac[i], &dd, &sc);
                            if (dd == d && sc == csec) A[m++] = (int)i;
                        }
                    } else {
                        for (int64_t a = a0; a < a1; ++a) {
                            int64_t dd; int sc;
                            dom_sector(c, &g, vac[keys[a].slot], &dd, &sc);
                            if (dd == d && sc == csec) A[m++] = (int)keys[a].slot;
                        }
                    }
                    if (m == 0) break;
                    for (int a = 0; a < m; ++a) {
                        double E[8];
                        ctr->clamps += vac_rates(c, &g, sp, vac[A[a]], Dp, E0, mlp, E, &G[8 * a]);
                        double sum = 0.0;
                        for (int k = 0; k < 8; ++k) sum = sum + G[8 * a + k];
                        R[a] = sum;
                    }
                    ctr->hop_evals += 8LL * m;
                    int P = 1, lev = 0;
                    double Rd = tree_build(R, m, buf, &P, &lev);
                    if (!(Rd > 0.0)) break;
                    double u_sel, u_t;
                    draw_uniforms(c->seed, it, (uint32_t)d, (uint32_t)p, (uint32_t)((uint64_t)p >> 32),
                                  &u_sel, &u_t);
                    double dt = (-orc_det_log(u_t)) / Rd;
                    if (t + dt > c->window_s) break;     /* overshooting draw discarded */
                    double r = u_sel * Rd;
                    int a = tree_descend(buf, R, m, P, &r);
                    int k = pick_hop(&G[8 * a], r);
                    apply_hop(&g, sp, vac, A[a], k);
                    t = t + dt;
                    it += 1;
                    ctr->events += 1;
                }
                a0 = a1;
            }
        }
        for (int64_t v = 0; v < c->n_voxels; ++v) clock[v] = clock[v] + c->window_s;
        *sweep_io = s + 1;
    }
    free(keys); free(A); free(R); free(G); free(buf);
    return ORC_OK;
}

/* entry: n = events per voxel (serial, domain == 0) or sweeps (sublattice).
 * vac[] holds global site indices in slot order (slot = rank of the initial site).
 * ctr_out[4] = events, hop_evals, terminal_voxels, clamps (accumulated). */
int orc_run(const orc_cfg* c, uint8_t* species, int64_t* vac, int64_t nvac, double* clock,
            int64_t* nev, int64_t* sweep, const double* eps, const double* E0, const double* mlp,
            int64_t n, int64_t* ctr_out)
{
    build_window();
    if (g_win_ready != 1) return ORC_INVALID;
    double Dp[2 * NSPEC * NSPEC];
    if (c->model == 0) {
        if (!eps || !E0) return ORC_INVALID;
        build_dp(eps, Dp);
    } else if (!mlp) {
        return ORC_INVALID;
    }
    orc_ctr ctr = {0, 0, 0, 0};
    int rc;
    if (c->domain[0] == 0)
        rc = run_serial(c, species, vac, nvac, clock, nev, Dp, E0, mlp, n, INFINITY, &ctr);
    else
        rc = run_sublattice(c, species, vac, nvac, clock, sweep, Dp, E0, mlp, n, &ctr);
    if (ctr_out) {
        ctr_out[0] += ctr.events; ctr_out[1] += ctr.hop_evals;
        ctr_out[2] += ctr.terminal_voxels; ctr_out[3] += ctr.clamps;
    }
    return rc;
}

/* serial mode: advance every voxel to the common physical time t_end (at most max_events events per
 * voxel); same counters as orc_run */
int orc_run_until(const orc_cfg* c, uint8_t* species, int64_t* vac, int64_t nvac, double* clock,
                  int64_t* nev, const double* eps, const double* E0, const double* mlp,
                  double t_end, int64_t max_events, int64_t* ctr_out)
{
    build_window();
    if (g_win_ready != 1 || c->domain[0] != 0) return ORC_INVALID;
    double Dp[2 * NSPEC * NSPEC];
    if (c->model == 0) {
        if (!eps || !E0) return ORC_INVALID;
        build_dp(eps, Dp);
    } else if (!mlp) {
        return ORC_INVALID;
    }
    orc_ctr ctr = {0, 0, 0, 0};
    int rc = run_serial(c, species, vac, nvac, clock, nev, Dp, E0, mlp, max_events, t_end, &ctr);
    if (ctr_out) {
        ctr_out[0] += ctr.events; ctr_out[1] += ctr.hop_evals;
        ctr_out[2] += ctr.terminal_voxels; ctr_out[3] += ctr.clamps;
    }
    return rc;
}

/* all rates of the current state, slot order: rates[i][8] (masked = 0), E[i][8] */
int orc_rates(const orc_cfg* c, const uint8_t* sp, const int64_t* vac, int64_t nvac,
              const double* eps, const double* E0, const double* mlp, double* rates, double* E)
{
    build_window();
    geom g = mk_geom(c);
    double Dp[2 * NSPEC * NSPEC];
    if (c->model == 0) build_dp(eps, Dp);
    int clamps = 0;
    for (int64_t i = 0; i < nvac; ++i) {
        double e[8], G[8];
        clamps += vac_rates(c, &g, sp, vac[i], Dp, E0, mlp, e, G);
        for (int k = 0; k < 8; ++k) {
            if (rates) rates[8 * i + k] = G[k];
            if (E) E[8 * i + k] = e[k];
        }
    }
    return clamps;
}

/* ------------------------------------------------------------------ */
/* world-model time mode (sec. V.A.1, sec. V.A.3)               */
/*   selection: the network outputs are the policy logits z_{i,k}; Eq. 1 masks infeasible hops and       */
/*     divides by tau_act; Eq. 2's global softmax over the competing set (the voxel, A15) picks (i, k)    */
/*     with probability exp(zhat)/sum exp(zhat) -- realised as the BKL tree/descent over the weights      */
/*     w = det_exp(min(zhat, 700)) (softmax is shift invariant, so no max subtraction is needed, W1)     */
/*   time: Eq. 7, dtau_hat = (u(s) - Gamma_tot(s)/Gamma_tot(s') u(s')) / Gamma_tot(s) with Gamma_tot   */
/*     from the physical (pair KRA) rates and u = uhat from the Poisson-time network on pooled windows   */
/*     (mean of the per-vacancy one-hot encodings, softplus head); the clock   */
/*     advances by max(dtau_hat, 1e-3 / Gamma_tot(s)) (S:409 floor, W4)                                 */
/* Readings W1-W6 are listed in DESIGN.md sec. 3.                                                       */
/* ------------------------------------------------------------------ */

/* softplus(y) = ln(1 + e^y), the Poisson network's non-negative head */
double orc_softplus(double y)
{
    if (y > 0.0) return y + orc_det_log(1.0 + orc_det_exp(-y));
    return orc_det_log(1.0 + orc_det_exp(y));
}

/* Eq. 7: the learned event-time increment; g_sp == 0 (s' has no event) -> u(s') term dropped */
double orc_delta_tau_hat(double u_s, double g_s, double u_sp, double g_sp)
{
    if (!(g_sp > 0.0)) return u_s / g_s;
    return (u_s - (g_s / g_sp) * u_sp) / g_s;
}

/* Poisson-time network on the pooled windows of n vacancies: x_f = count_f / n over the one-hot features
 * f = 7*slot + species; h_j = ReLU(bt1_j + sum_f x_f Wt1[f][j]) (dense fma loop in f order); y = bt2 +
 * sum_j h_j wt2_j; uhat = softplus(y).  tnet = Wt1[448*H], bt1[H], wt2[H], bt2[1]. */
double orc_poisson_net(const uint8_t* sigmas /* [n][64] */, int n, const double* tnet, int H)
{
    if (n <= 0) return 0.0;
    const double* Wt1 = tnet;
    const double* bt1 = Wt1 + 448 * (size_t)H;
    const double* wt2 = bt1 + H;
    const double* bt2 = wt2 + H;
    int cnt[448];
    memset(cnt, 0, sizeof(cnt));
    for (int i = 0; i < n; ++i)
        for (int s = 0; s < NWIN; ++s) cnt[7 * s + sigmas[(size_t)i * NWIN + s]] += 1;
    double y = bt2[0];
    for (int j = 0; j < H; ++j) {
        double acc = bt1[j];
        for (int f = 0; f < 448; ++f) {
            double x = (double)cnt[f] / (double)n;
            acc = fma(x, Wt1[(size_t)f * H + j], acc);
        }
        double h = acc > 0.0 ? acc : 0.0;
        y = fma(h, wt2[j], y);
    }
    return orc_softplus(y);
}

typedef struct { const double* tnet; int H; double tau; } world_par;

/* policy weights W[m][8], physical rates G[m][8] (pair KRA, the voxel's T) of the m members of a voxel, their
 * trees' totals, and uhat of the voxel's pooled windows */
static void world_eval(const orc_cfg* c, const geom* g, const uint8_t* sp, const int64_t* vac, const int* members,
                       int m, const double* Dp, const double* E0, const double* mlp, const world_par* wp,
                       double* W, double* G, double* Rw, double* Rg, double* buf, uint8_t* sig,
                       double* wtot, double* gtot, double* uhat, int* P_out)
{
    orc_cfg cp = *c;
    cp.model = 0;                                  /* physical rates: pair KRA */
    for (int a = 0; a < m; ++a) {
        int64_t vsite = vac[members[a]];
        double E[8], z[8];
        vac_rates(&cp, g, sp, vsite, Dp, E0, NULL, E, &G[8 * a]);
        window_of(g, sp, vsite, &sig[(size_t)a * NWIN]);
        mlp_forward(&sig[(size_t)a * NWIN], mlp, z);
        double sw = 0.0, sg = 0.0;
        for (int k = 0; k < 8; ++k) {
            double w = 0.0;
            if (sig[(size_t)a * NWIN + k] != VAC) {                     /* Eq. 1 mask m_{i,k} */
                double zh = z[k] / wp->tau;
                if (zh > 700.0) zh = 700.0;
                w = orc_det_exp(zh);
            }
            W[8 * a + k] = w;
            sw = sw + w;
            sg = sg + G[8 * a + k];
        }
        Rw[a] = sw;
        Rg[a] = sg;
    }
    int P = 1, lev = 0;
    *gtot = (m > 0) ? tree_build(Rg, m, buf, &P, &lev) : 0.0;
    *wtot = (m > 0) ? tree_build(Rw, m, buf, &P, &lev) : 0.0;     /* buf keeps the policy tree */
    *P_out = P;
    *uhat = orc_poisson_net(sig, m, wp->tnet, wp->H);
}

/* serial world-model steps: n events per voxel (or until no feasible event); same Philox counters as BKL */
int orc_run_world(const orc_cfg* c, uint8_t* sp, int64_t* vac, int64_t nvac, double* clock, int64_t* nev,
                  const double* eps, const double* E0, const double* mlp, const double* tnet, int H, double tau_act,
                  int64_t n, int64_t* ctr_out)
{
    build_window();
    if (g_win_ready != 1 || c->domain[0] != 0 || !eps || !E0 || !mlp || !tnet || H < 1 || !(tau_act > 0.0))
        return ORC_INVALID;
    double Dp[2 * NSPEC * NSPEC];
    build_dp(eps, Dp);
    geom g = mk_geom(c);
    world_par wp = {tnet, H, tau_act};
    int* members = (int*)malloc(sizeof(int) * (size_t)(nvac + 1));
    double* W = (double*)malloc(sizeof(double) * 8 * (size_t)(nvac + 1));
    double* G = (double*)malloc(sizeof(double) * 8 * (size_t)(nvac + 1));
    double* Rw = (double*)malloc(sizeof(double) * (size_t)(nvac + 1));
    double* Rg = (double*)malloc(sizeof(double) * (size_t)(nvac + 1));
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)(nvac + 2));
    uint8_t* sig = (uint8_t*)malloc((size_t)NWIN * (size_t)(nvac + 1));
    int rc = ORC_OK;
    orc_ctr ctr = {0, 0, 0, 0};
    for (int64_t v = 0; v < c->n_voxels; ++v) {
        int m = 0;
        for (int64_t i = 0; i < nvac; ++i)
            if (vac[i] / g.sites_per_voxel == v) members[m++] = (int)i;
        double wtot, gtot, uhat;
        int P;
        world_eval(c, &g, sp, vac, members, m, Dp, E0, mlp, &wp, W, G, Rw, Rg, buf, sig, &wtot, &gtot, &uhat, &P);
        for (int64_t e = 0; e < n; ++e) {
            ctr.hop_evals += 8LL * m;
            if (!(wtot > 0.0) || !(gtot > 0.0)) { ctr.terminal_voxels += 1; rc = ORC_TERMINAL; break; }
            double u_sel, u_t;
            draw_uniforms(c->seed, (uint32_t)nev[v], (uint32_t)((uint64_t)nev[v] >> 32), (uint32_t)v, 0u, &u_sel, &u_t);
            double r = u_sel * wtot;
            int a = tree_descend(buf, Rw, m, P, &r);
            int k = pick_hop(&W[8 * a], r);
            apply_hop(&g, sp, vac, members[a], k);
            const double u_s = uhat, g_s = gtot;
            world_eval(c, &g, sp, vac, members, m, Dp, E0, mlp, &wp, W, G, Rw, Rg, buf, sig, &wtot, &gtot, &uhat, &P);
            double dt = orc_delta_tau_hat(u_s, g_s, uhat, gtot);
            double fl = 1e-3 / g_s;
            clock[v] = clock[v] + (dt > fl ? dt : fl);
            nev[v] += 1;
            ctr.events += 1;
        }
    }
    free(members); free(W); free(G); free(Rw); free(Rg); free(buf); free(sig);
    if (ctr_out) {
        ctr_out[0] += ctr.events; ctr_out[1] += ctr.hop_evals;
        ctr_out[2] += ctr.terminal_voxels; ctr_out[3] += ctr.clamps;
    }
    return rc;
}

/* the world-model quantities of one voxel's current state (pins): policy weights W[m][8], physical rates
 * G[m][8] (slot order of the voxel's members), their totals and uhat */
int orc_world_eval(const orc_cfg* c, const uint8_t* sp, const int64_t* vac, int64_t nvac, int64_t vox,
                   const double* eps, const double* E0, const double* mlp, const double* tnet, int H, double tau_act,
                   double* W, double* G, double* out3 /* wtot, gtot, uhat */)
{
    build_window();
    double Dp[2 * NSPEC * NSPEC];
    build_dp(eps, Dp);
    geom g = mk_geom(c);
    world_par wp = {tnet, H, tau_act};
    int* members = (int*)malloc(sizeof(int) * (size_t)(nvac + 1));
    int m = 0;
    for (int64_t i = 0; i < nvac; ++i)
        if (vac[i] / g.sites_per_voxel == vox) members[m++] = (int)i;
    double* Rw = (double*)malloc(sizeof(double) * (size_t)(m + 1));
    double* Rg = (double*)malloc(sizeof(double) * (size_t)(m + 1));
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)(m + 2));
    uint8_t* sig = (uint8_t*)malloc((size_t)NWIN * (size_t)(m + 1));
    int P;
    world_eval(c, &g, sp, vac, members, m, Dp, E0, mlp, &wp, W, G, Rw, Rg, buf, sig, &out3[0], &out3[1], &out3[2], &P);
    free(members); free(Rw); free(Rg); free(buf); free(sig);
    return m;
}

/* ------------------------------------------------------------------ */
/* statistics: Cu clusters under 1NN adjacency per voxel    */
/* out[0..5] = n_cu, n_clusters(>=1), n_clusters(>=2), largest, monomers,
 *             precipitates(>= nstar); out[6] = mean size of clusters >= 2;
 *             out[7] = Cu-Cu 1NN bond count (for alpha_1); hist[size] counts  */
/* ------------------------------------------------------------------ */
int orc_cluster_stats(const orc_cfg* c, const uint8_t* sp, int64_t vox, int cu, int nstar,
                      double* out, int64_t* hist, int64_t hist_len)
{
    geom g = mk_geom(c);
    int64_t N = g.sites_per_voxel;
    int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    uint8_t* seen = (uint8_t*)calloc((size_t)N, 1);
    int64_t ncu = 0, ncl = 0, ncl2 = 0, largest = 0, mono = 0, prec = 0, sum2 = 0, bonds = 0;
    if (hist) memset(hist, 0, sizeof(int64_t) * (size_t)hist_len);
    for (int64_t i = 0; i < N; ++i) {
        int64_t site = vox * N + i;
        if (sp[site] != cu) continue;
        ++ncu;
        int64_t vv; int p[3];
        site_pos(&g, site, &vv, p);
        for (int j = 0; j < 8; ++j) {
            int q[3] = {p[0] + NN1[j][0], p[1] + NN1[j][1], p[2] + NN1[j][2]};
            if (sp[pos_site(&g, vox, q)] == cu) ++bonds;
        }
        if (seen[i]) continue;
        int64_t top = 0, size = 0;
        stack[top++] = i; seen[i] = 1;
        while (top > 0) {
            int64_t cur = stack[--top];
            ++size;
            int64_t v2; int pc[3];
            site_pos(&g, vox * N + cur, &v2, pc);
            for (int j = 0; j < 8; ++j) {
                int q[3] = {pc[0] + NN1[j][0], pc[1] + NN1[j][1], pc[2] + NN1[j][2]};
                int64_t t = pos_site(&g, vox, q) - vox * N;
                if (!seen[t] && sp[vox * N + t] == cu) { seen[t] = 1; stack[top++] = t; }
            }
        }
        ++ncl;
        if (size >= 2) { ++ncl2; sum2 += size; }
        if (size == 1) ++mono;
        if (size >= nstar) ++prec;
        if (size > largest) largest = size;
        if (hist && size < hist_len) hist[size] += 1;
    }
    out[0] = (double)ncu; out[1] = (double)ncl; out[2] = (double)ncl2; out[3] = (double)largest;
    out[4] = (double)mono; out[5] = (double)prec;
    out[6] = ncl2 > 0 ? (double)sum2 / (double)ncl2 : 0.0;
    out[7] = (double)(bonds / 2);
    free(stack); free(seen);
    return 0;
}
