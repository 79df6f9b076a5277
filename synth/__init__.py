"""Seeded synthetic inputs for the AKMC hot path (shared by the CUDA path and the oracle as DATA).

This module holds none of the method's arithmetic (no barriers, rates, selection).
It produces: lattices (species bytes), vacancy placements, illustrative pair
parameters, barrier-network weights and the configuration presets C1..C5 of
BASELINE.json.  Recipes are stated in DESIGN.md sec. 4 and cite:

* A508-3 composition P:533 (sec. VI.B), folded to Fe-Cu-Ni-Mn-Si at.%
* random ideal solid solution, largest-remainder counts, no V-V 1NN at t=0 (A24)
* illustrative pair energies ("defaults ... documented as illustrative")
* physics-embedded MLP weights (48 gate units reproduce the
  Fe-referenced pair KRA barrier; A9), optional seeded residual, or fully random
  weights

Geometry here (window offsets, neighbour tables) is an independent numpy
implementation used only to build the physics-embedded weights.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SPECIES = ("Fe", "Cu", "Ni", "Mn", "Si", "P", "V")
FE, CU, NI, MN, SI, P_, VAC = range(7)
NSPEC = 7
NHID = 256
KB_EV = 8.617333262e-5
NU0 = 6.0e12
T_DEFAULT = 563.0               # A13
A0_ANGSTROM = 2.866
CUTOFF_ANGSTROM = 6.0

# ---------------------------------------------------------------------------
# composition: wt.% -> at.%, trace species folded into Fe
# ---------------------------------------------------------------------------
_A508_WT = {"C": 0.167, "Si": 0.193, "Mn": 1.35, "S": 0.002, "P": 0.005, "Cr": 0.086,
            "Ni": 0.738, "Cu": 0.027, "Mo": 0.481, "V": 0.007}
_MASS = {"Fe": 55.845, "C": 12.011, "Si": 28.085, "Mn": 54.938, "S": 32.06, "P": 30.974,
         "Cr": 51.996, "Ni": 58.693, "Cu": 63.546, "Mo": 95.95, "V": 50.942}


def a508_atomic_fractions() -> dict:
    """A508-3 in at.%, with C, S, Cr, Mo, V, P folded into Fe (fractions of atoms)."""
    wt = dict(_A508_WT)
    wt["Fe"] = 100.0 - sum(wt.values())
    mol = {k: v / _MASS[k] for k, v in wt.items()}
    tot = sum(mol.values())
    at = {k: v / tot for k, v in mol.items()}
    folded = {"Fe": at["Fe"] + at["C"] + at["S"] + at["Cr"] + at["Mo"] + at["V"] + at["P"],
              "Cu": at["Cu"], "Ni": at["Ni"], "Mn": at["Mn"], "Si": at["Si"]}
    return folded


def largest_remainder_counts(fractions: dict, n: int) -> np.ndarray:
    """Integer species counts summing to n by largest remainder."""
    f = np.zeros(NSPEC - 1)
    for k, v in fractions.items():
        f[SPECIES.index(k)] = v
    f = f / f.sum()
    raw = f * n
    base = np.floor(raw).astype(np.int64)
    rem = n - int(base.sum())
    order = np.argsort(-(raw - base), kind="stable")
    base[order[:rem]] += 1
    return base


# ---------------------------------------------------------------------------
# lattices
# ---------------------------------------------------------------------------
_NN1_HALF = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], dtype=np.int64)


def _site_to_pos(idx: np.ndarray, L):
    b = idx & 1
    cell = idx >> 1
    x = cell % L[0]
    y = (cell // L[0]) % L[1]
    z = cell // (L[0] * L[1])
    return 2 * x + b, 2 * y + b, 2 * z + b


def _pos_to_site(px, py, pz, L):
    px = px % (2 * L[0]); py = py % (2 * L[1]); pz = pz % (2 * L[2])
    return 2 * ((px >> 1) + L[0] * ((py >> 1) + L[1] * (pz >> 1))) + (px & 1)


def make_voxel(cells, fractions: dict, n_vac: int, rng: np.random.Generator) -> np.ndarray:
    """One periodic voxel: random ideal solid solution with exact (largest-remainder)
    counts over the sites - n_vac atoms, then n_vac vacancies placed uniformly with no
    V-V 1NN pair (A24).  Canonical site index 2*(x + Lx*(y + Ly*z)) + b."""
    L = tuple(int(c) for c in cells)
    n = 2 * L[0] * L[1] * L[2]
    if n_vac > 0.01 * n:
        raise ValueError("n_vac exceeds 1% of sites (S:48)")
    counts = largest_remainder_counts(fractions, n - n_vac)
    sp = np.repeat(np.arange(NSPEC - 1, dtype=np.uint8), counts)
    sp = np.concatenate([sp, np.full(n_vac, VAC, dtype=np.uint8)])
    # place the atoms by a seeded permutation of the non-vacancy sites: choose vacancy
    # sites first (uniform, rejecting 1NN conflicts), then shuffle atoms into the rest.
    chosen = []
    taken = set()
    while len(chosen) < n_vac:
        s = int(rng.integers(0, n))
        if s in taken:
            continue
        px, py, pz = _site_to_pos(np.array([s]), L)
        nb = _pos_to_site(px + _NN1_HALF[:, 0], py + _NN1_HALF[:, 1], pz + _NN1_HALF[:, 2], L)
        if any(int(t) in taken for t in nb):
            continue
        chosen.append(s)
        taken.add(s)
    out = np.empty(n, dtype=np.uint8)
    mask = np.ones(n, dtype=bool)
    if n_vac:
        mask[np.array(chosen, dtype=np.int64)] = False
    atoms = sp[: n - n_vac].copy()
    rng.shuffle(atoms)
    out[mask] = atoms
    out[~mask] = VAC
    return out


def make_lattice(cells, n_voxels: int, fractions: dict, n_vac_per_voxel: int, seed: int) -> np.ndarray:
    """n_voxels independent voxels, seeded with NumPy PCG64(seed), concatenated."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.concatenate([make_voxel(cells, fractions, n_vac_per_voxel, rng) for _ in range(n_voxels)])


def make_lattice_iid(cells, fractions: dict, n_vac: int, seed: int, device=None):
    """Large-lattice recipe (C3/C5): species i.i.d. per site with the composition's
    probabilities (multinomial counts), then n_vac vacancies at distinct uniform sites
    (V-V 1NN pairs not excluded; expected count ~ 4*n_vac*c_v).  Generated with torch on
    `device` (plumbing only).  Returns a torch uint8 tensor."""
    import torch
    L = tuple(int(c) for c in cells)
    n = 2 * L[0] * L[1] * L[2]
    g = torch.Generator(device=device or "cpu")
    g.manual_seed(int(seed))
    f = np.zeros(NSPEC - 1)
    for k, v in fractions.items():
        f[SPECIES.index(k)] = v
    cdf = np.cumsum(f / f.sum())
    out = torch.empty(n, dtype=torch.uint8, device=device)
    chunk = 1 << 27
    thr = torch.tensor(cdf[:-1], dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        u = torch.rand(e - s, generator=g, device=device)
        out[s:e] = torch.bucketize(u, thr, right=True).to(torch.uint8)
    if n_vac:
        idx = torch.randint(0, n, (int(n_vac * 1.05) + 64,), generator=g, device=device)
        idx = torch.unique(idx)
        perm = torch.randperm(idx.numel(), generator=g, device=device)
        idx = idx[perm[:n_vac]]
        out[idx] = VAC
    return out


# ---------------------------------------------------------------------------
# illustrative pair parameters (declared illustrative, not fitted)
# ---------------------------------------------------------------------------
def illustrative_pair_params():
    """eps[2][7][7] (eV), symmetric; E0[7] (eV).  Magnitudes follow SURVEY A.11/A.14
    (1NN ~ -0.78 eV, 2NN ~ half, vacancy bonds ~ -0.2 eV).  NOT from the paper."""
    e1 = np.array([
        # Fe      Cu      Ni      Mn      Si      P       V
        [-0.778, -0.759, -0.790, -0.770, -0.800, -0.760, -0.200],
        [-0.759, -0.816, -0.780, -0.745, -0.770, -0.740, -0.180],
        [-0.790, -0.780, -0.805, -0.785, -0.810, -0.775, -0.210],
        [-0.770, -0.745, -0.785, -0.765, -0.790, -0.755, -0.230],
        [-0.800, -0.770, -0.810, -0.790, -0.760, -0.770, -0.250],
        [-0.760, -0.740, -0.775, -0.755, -0.770, -0.720, -0.260],
        [-0.200, -0.180, -0.210, -0.230, -0.250, -0.260, -0.100],
    ])
    e2 = 0.5 * e1
    eps = np.stack([e1, e2]).astype(np.float64)
    assert np.array_equal(eps, np.transpose(eps, (0, 2, 1)))
    E0 = np.array([0.62, 0.54, 0.68, 0.60, 0.78, 0.70, 0.0], dtype=np.float64)
    return eps, E0


# ---------------------------------------------------------------------------
# barrier-network weights (one-hot 448 -> 256 -> 256 -> 8, ReLU)
# flat layout: W1[448*256] (row f = 7*slot + species), b1[256], W2[256*256] (row = input),
#              b2[256], W3[256*8], b3[8]
# ---------------------------------------------------------------------------
MLP_SIZE = 448 * NHID + NHID + NHID * NHID + NHID + NHID * 8 + 8


def window_offsets_np() -> np.ndarray:
    """64 half-cell offsets within 6.0 A (a0 = 2.866 A), sorted by (|h|^2, hx, hy, hz)."""
    rows = []
    for hx in range(-5, 6):
        for hy in range(-5, 6):
            for hz in range(-5, 6):
                if len({hx & 1, hy & 1, hz & 1}) != 1 or (hx, hy, hz) == (0, 0, 0):
                    continue
                h2 = hx * hx + hy * hy + hz * hz
                if math.sqrt(h2) * A0_ANGSTROM / 2 <= CUTOFF_ANGSTROM:
                    rows.append((h2, hx, hy, hz))
    rows.sort()
    return np.array([r[1:] for r in rows], dtype=np.int64)


def split_mlp(mlp: np.ndarray):
    o = 0
    W1 = mlp[o:o + 448 * NHID].reshape(448, NHID); o += 448 * NHID
    b1 = mlp[o:o + NHID]; o += NHID
    W2 = mlp[o:o + NHID * NHID].reshape(NHID, NHID); o += NHID * NHID
    b2 = mlp[o:o + NHID]; o += NHID
    W3 = mlp[o:o + NHID * 8].reshape(NHID, 8); o += NHID * 8
    b3 = mlp[o:o + 8]
    return W1, b1, W2, b2, W3, b3


def pack_mlp(W1, b1, W2, b2, W3, b3) -> np.ndarray:
    return np.concatenate([np.asarray(a, dtype=np.float64).ravel() for a in (W1, b1, W2, b2, W3, b3)])


def physics_mlp(eps, E0, gate_c: float = 2.0, residual: float = 0.0, seed: int = 0) -> np.ndarray:
    """Physics-embedded weights (reading A9).

    Unit u = 6k + x (k = hop 0..7, x = non-vacancy species 0..5):
      pre_u = E0[x] - C + C*[sigma_k == x] + 1/2 sum_{slot j, species y} w_{k,x}[j][y] [sigma_j == y]
    with w_{k,x}[j][y] = sum_s (a_k[s][j] - b_k[s][j]) Dp[s][x][y], a_k = shell-s neighbours of the
    vacancy except n_k, b_k = shell-s neighbours of n_k except the vacancy, and the Fe-referenced
    Dp[s][x][y] = (eps[s][x][y]-eps[s][V][y]) - (eps[s][x][Fe]-eps[s][V][Fe]).  ReLU(pre_u) = E_k when
    sigma_k == x, else 0 (for C large enough).  Layer 2 = identity on the 48 units; layer 3 sums
    over x.  Units 48..255 carry an optional seeded residual (perturbation of the barriers)."""
    eps = np.asarray(eps, dtype=np.float64)
    E0 = np.asarray(E0, dtype=np.float64)
    off = window_offsets_np()
    h2 = (off ** 2).sum(1)
    shell_of = {3: 0, 4: 1}
    Dp = np.zeros((2, NSPEC, NSPEC))
    for s in range(2):
        for x in range(NSPEC):
            for y in range(NSPEC):
                Dp[s, x, y] = (eps[s, x, y] - eps[s, VAC, y]) - (eps[s, x, FE] - eps[s, VAC, FE])
    W1 = np.zeros((64, NSPEC, NHID))
    b1 = np.zeros(NHID)
    for k in range(8):
        ek = off[k]
        coef = np.zeros((64, 2))           # coef[j][s] = a_k[s][j] - b_k[s][j]
        for j in range(64):
            if j != k and h2[j] in shell_of:
                coef[j, shell_of[h2[j]]] += 1.0
            d = off[j] - ek
            dd = int((d ** 2).sum())
            if dd in shell_of:
                coef[j, shell_of[dd]] -= 1.0
        for x in range(NSPEC - 1):
            u = 6 * k + x
            for j in range(64):
                for y in range(NSPEC):
                    W1[j, y, u] = 0.5 * (coef[j, 0] * Dp[0, x, y] + coef[j, 1] * Dp[1, x, y])
            W1[k, x, u] += gate_c
            b1[u] = E0[x] - gate_c
    W2 = np.zeros((NHID, NHID)); b2 = np.zeros(NHID)
    W3 = np.zeros((NHID, 8)); b3 = np.zeros(8)
    for k in range(8):
        for x in range(NSPEC - 1):
            W2[6 * k + x, 6 * k + x] = 1.0
            W3[6 * k + x, k] = 1.0
    if residual > 0.0:
        rng = np.random.Generator(np.random.PCG64(seed))
        W1[:, :, 48:] = rng.normal(0.0, 0.05, size=(64, NSPEC, NHID - 48))
        b1[48:] = 0.1
        W2[48:, 48:] = rng.normal(0.0, 1.0 / 16.0, size=(NHID - 48, NHID - 48))
        b2[48:] = 0.05
        W3[48:, :] = rng.normal(0.0, residual, size=(NHID - 48, 8))
    return pack_mlp(W1.reshape(448, NHID), b1, W2, b2, W3, b3)


def random_mlp(seed: int, s1: float = 0.05, s2: float = 1.0 / 16.0, s3: float = 0.02,
               out_bias: float = 0.6) -> np.ndarray:
    """Fully random weights: W ~ N(0, s), output ~0.4-0.9 eV."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W1 = rng.normal(0.0, s1, size=(448, NHID)); b1 = rng.normal(0.05, 0.05, size=NHID)
    W2 = rng.normal(0.0, s2, size=(NHID, NHID)); b2 = rng.normal(0.0, 0.05, size=NHID)
    W3 = rng.normal(0.0, s3, size=(NHID, 8)); b3 = np.full(8, out_bias)
    return pack_mlp(W1, b1, W2, b2, W3, b3)


def policy_mlp(mlp: np.ndarray, kT: float) -> np.ndarray:
    """World-model policy weights from a barrier network (reading W2): the last layer scaled
    by -1/kT, so the raw outputs are the logits z_k = -E_k/kT and Eq. 2's softmax selects hops with the BKL
    probabilities Gamma_a / Gamma_tot (nu0 cancels in the softmax)."""
    W1, b1, W2, b2, W3, b3 = (a.copy() for a in split_mlp(np.asarray(mlp, dtype=np.float64)))
    return pack_mlp(W1, b1, W2, b2, W3 * (-1.0 / kT), b3 * (-1.0 / kT))


def poisson_net(seed: int, H: int = 32, s1: float = 0.3, s2: float = 0.5, bias: float = 0.5) -> np.ndarray:
    """Synthetic Poisson-time network (no trained weights exist, P:557-563 OUT): Wt1[448*H], bt1[H], wt2[H],
    bt2[1] with uhat = softplus(...) = O(1) (SPEC S:337-340 shape, reading W3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    Wt1 = rng.normal(0.0, s1, size=(448, H)); bt1 = rng.normal(0.1, 0.1, size=H)
    wt2 = rng.normal(0.0, s2, size=H); bt2 = np.array([bias])
    return np.concatenate([Wt1.ravel(), bt1, wt2, bt2])


# ---------------------------------------------------------------------------
# windows and presets
# ---------------------------------------------------------------------------
def window_seconds(lam: float, E0_fe: float, T: float = T_DEFAULT, nu0: float = NU0, kB: float = KB_EV) -> float:
    """Delta_win = lambda / (8 nu0 exp(-E0[Fe]/kB T)) (reading A22)."""
    return lam / (8.0 * nu0 * math.exp(-E0_fe / (kB * T)))


def voxel_temperatures(n: int, seed: int, lo: float = 558.0, hi: float = 577.0) -> np.ndarray:
    """Per-voxel temperatures for the C4 heterogeneous-T variant (uniform in 558-577 K)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, size=n)


def random_windows(n: int, seed: int, solute: float = 0.3, vac: float = 0.02) -> np.ndarray:
    """Random 64-slot windows (uint8 species codes) for network-precision studies:
    each slot is V with prob `vac`, else a solute (Cu..P uniform) with prob `solute`, else Fe."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random((n, 64))
    w = np.zeros((n, 64), dtype=np.uint8)
    sol = rng.integers(1, 6, size=(n, 64)).astype(np.uint8)
    w[u < solute] = sol[u < solute]
    w[u < vac] = VAC
    return w


@dataclass
class Preset:
    name: str
    cells: tuple
    n_voxels: int
    n_vac_per_voxel: int
    fractions: dict
    domain: tuple = (0, 0, 0)
    lam: float = 0.25
    seed: int = 2604
    notes: str = ""
    extra: dict = field(default_factory=dict)


def fe_cu_fractions(cu_at: float = 0.01) -> dict:
    return {"Fe": 1.0 - cu_at, "Cu": cu_at}


def preset(name: str) -> Preset:
    """BASELINE.json configs C1..C5; PCG64 seed = 2604 + config index."""
    rpv = a508_atomic_fractions()
    if name == "C1":
        return Preset("C1", (16, 16, 16), 1, 1, fe_cu_fractions(0.01), seed=2605,
                      notes="Fe-1at%Cu 16^3, 1 V, serial BKL")
    if name == "C2":
        return Preset("C2", (64, 64, 64), 1, 10, rpv, seed=2606, notes="RPV 64^3, 10 V, serial BKL")
    if name == "C3":
        return Preset("C3", (512, 512, 512), 1, 26844, rpv, domain=(8, 8, 8), seed=2607,
                      notes="RPV 512^3, c_v 1e-4, sublattice D=8, lambda=1/4")
    if name == "C4":
        return Preset("C4", (64, 64, 64), 4096, 10, rpv, seed=2608,
                      notes="4096 voxels of 64^3 (512 per GPU), 10 V each, serial BKL per voxel")
    if name == "C5":
        return Preset("C5", (1024, 1024, 1024), 1, 214748, rpv, domain=(8, 8, 8), seed=2609,
                      notes="1024^3 per GPU, c_v 1e-4, sublattice D=8, lambda=1/4")
    raise KeyError(name)


def with_vacancy_cluster(species: np.ndarray, cells, center) -> tuple:
    """Degenerate input: a vacancy at basis-0 site `center` = (x, y, z) whose eight first neighbours are
    also vacancies (the basis-1 sites of cells x-1..x, y-1..y, z-1..z with basis 1 at +(1/2, 1/2, 1/2)).
    Every hop of the centre is masked (m_k = 0, P:288-289 / A14), so its R_i = 0 leaf sits inside the
    competing set.  Returns (species copy, centre site id).  Geometry only, none of the method's arithmetic."""
    Lx, Ly, Lz = cells
    x, y, z = center
    sp = np.array(species, dtype=np.uint8, copy=True)

    def site(cx, cy, cz, b):
        return 2 * ((cx % Lx) + Lx * ((cy % Ly) + Ly * (cz % Lz))) + b

    c = site(x, y, z, 0)
    sp[c] = 6
    for dx in (-1, 0):
        for dy in (-1, 0):
            for dz in (-1, 0):
                sp[site(x + dx, y + dy, z + dz, 1)] = 6
    return sp, c
