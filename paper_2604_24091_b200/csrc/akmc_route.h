// akmc_route.h -- routing rules of the per-phase halo-delta exchange (C5; sec. V.B.3),
// plain C++ usable from host code (tests/test_route_cpu.py compiles it with g++) and device code.
//
// An entry is a site written in the last phase (species write) or a vacancy that left its block (migration), at
// global cell g.  Its destinations: every rank whose EXTENDED region (block + kHalo cells per decomposed face)
// contains g (species), or the one rank whose block contains g (migration).
//  * direct exchange: the writer sends the entry to each destination (up to 26 neighbour blocks; 7 distinct
//    ranks on a 2x2x2 torus);
//  * shift exchange (the paper's communication scheme): stages along the decomposed axes in order x, y, z; at
//    stage a a holder with block coordinates P sends to its neighbour at P_a + d (d = +-1) iff g lies in that
//    neighbour's range along a AND in P's own range along every earlier stage's axis b < a.  Receivers keep the
//    entry for the later stages, so edge and corner destinations are reached in <= 3 hops with 2 messages per
//    axis (6 instead of 26).  With 2 ranks along an axis both neighbours are one rank: one message, d = +1.
#pragma once

#ifdef __CUDACC__
#define AKMC_HD __host__ __device__ __forceinline__
#else
#define AKMC_HD inline
#endif

namespace akmc {
namespace route {

AKMC_HD int pmod(int a, int m)
{
    const int r = a % m;
    return r < 0 ? r + m : r;
}

// along one axis: is global cell gc in the extended range (halo h) / the owned block of the block at coordinate c?
AKMC_HD bool in_ext_axis(int gc, int c, int L, int h, int G) { return pmod(gc - c * L + h, G) < L + 2 * h; }
AKMC_HD bool in_blk_axis(int gc, int c, int L, int G) { return pmod(gc - c * L, G) < L; }

AKMC_HD bool in_range(int gc, int c, int L, int h, int G, bool migrate)
{
    return migrate ? in_blk_axis(gc, c, L, G) : in_ext_axis(gc, c, L, h, G);
}

// shift stage a: does the holder at block coordinates P send the entry at global cell g to its neighbour P_a + d?
AKMC_HD bool shift_send(const int g[3], const int P[3], int a, int d, const int L[3], const int grid[3], int h, bool migrate)
{
    for (int b = 0; b < a; ++b)
        if (grid[b] > 1 && !in_range(g[b], P[b], L[b], h, grid[b] * L[b], migrate)) return false;
    const int c = pmod(P[a] + d, grid[a]);
    return in_range(g[a], c, L[a], h, grid[a] * L[a], migrate);
}

// the distinct neighbour directions of axis a: +1 and -1, or only +1 when two ranks share the axis
AKMC_HD int shift_dirs(int grid_a) { return grid_a > 2 ? 2 : (grid_a == 2 ? 1 : 0); }

} // namespace route
} // namespace akmc
