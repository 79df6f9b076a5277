"""Host logic of the C5 halo-delta exchange (sec. V.B.3), -m "not gpu":
the product's routing header (csrc/akmc_route.h) compiled with g++ and driven on virtual rank grids.

* shift == direct: for random species writes and vacancy migrations near block faces, edges and corners, the
  staged X -> Y -> Z forwarding delivers every entry to exactly the ranks the direct exchange sends it to
  (species: every rank whose extended region holds the site; migration: exactly one arrival, at the owner);
* message counts per rank and phase ("6 vs 26"): 3x3x3 grid -> shift 6, direct 26 distinct peers;
  2x2x2 -> 3 vs 7; 2x2x1 -> 2 vs 3; 2x1x1 -> 1 vs 1.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_24091_b200", "csrc")

DRIVER = r'''
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>
#include <random>
#include "akmc_route.h"
using namespace akmc::route;
int main(int argc, char** argv) {
    int grid[3] = {atoi(argv[1]), atoi(argv[2]), atoi(argv[3])};
    const int L[3] = {12, 10, 14}, h = 2;
    const int G[3] = {grid[0] * L[0], grid[1] * L[1], grid[2] * L[2]};
    auto rid = [&](const int c[3]) { return c[0] + grid[0] * (c[1] + grid[1] * c[2]); };
    auto coords = [&](int r, int c[3]) { c[0] = r % grid[0]; c[1] = (r / grid[0]) % grid[1]; c[2] = r / (grid[0] * grid[1]); };
    const int nr = grid[0] * grid[1] * grid[2];
    std::mt19937 rng(7);
    long bad = 0, checked = 0;
    for (int t = 0; t < 200000; ++t) {
        int S[3]; coords(rng() % nr, S);
        const bool mig = (rng() % 3) == 0;
        int g[3];
        for (int a = 0; a < 3; ++a) {
            // a cell of S's block or one cell outside it (a hop reaches half a cell), biased to faces/edges/corners
            int off = (rng() % 4 == 0) ? (int)(rng() % L[a]) : (int)(rng() % 4) - 1;
            if (rng() % 2) off = L[a] - 1 - off;
            if (grid[a] == 1) off = pmod(off, L[a]);
            g[a] = pmod(S[a] * L[a] + off, G[a]);
        }
        // direct destinations
        std::multiset<int> want;
        for (int r = 0; r < nr; ++r) {
            if (r == rid(S)) continue;
            int c[3]; coords(r, c);
            bool in = true;
            for (int a = 0; a < 3; ++a) if (grid[a] > 1 && !in_range(g[a], c[a], L[a], h, G[a], mig)) in = false;
            if (in) want.insert(r);
        }
        if (mig) {   // a migration exists only when the vacancy left S's block
            bool inS = true;
            for (int a = 0; a < 3; ++a) if (grid[a] > 1 && !in_blk_axis(g[a], S[a], L[a], G[a])) inS = false;
            if (inS) continue;
        }
        // shift simulation
        std::vector<int> holders = {rid(S)};
        std::multiset<int> got;
        for (int a = 0; a < 3; ++a) {
            if (grid[a] == 1) continue;
            std::vector<int> recv;
            for (int P : holders) {
                int c[3]; coords(P, c);
                for (int k = 0; k < shift_dirs(grid[a]); ++k) {
                    const int d = k == 0 ? 1 : -1;
                    if (!shift_send(g, c, a, d, L, grid, h, mig)) continue;
                    int q[3] = {c[0], c[1], c[2]}; q[a] = pmod(c[a] + d, grid[a]);
                    recv.push_back(rid(q));
                }
            }
            for (int r : recv) { holders.push_back(r); got.insert(r); }
        }
        // keep only receivers that need it (species: in their extended region; migration: owner)
        std::multiset<int> used;
        for (int r : got) if (want.count(r)) used.insert(r);
        std::set<int> wu(want.begin(), want.end()), uu(used.begin(), used.end());
        ++checked;
        if (wu != uu) ++bad;
        if (mig) { for (int r : wu) if (used.count(r) != 1) ++bad; }   // exactly one arrival at the owner
    }
    // message counts per rank: shift = sum over decomposed axes of distinct neighbours; direct = distinct peers
    int shift_msgs = 0;
    for (int a = 0; a < 3; ++a) shift_msgs += shift_dirs(grid[a]);
    std::set<int> peers;
    int c0[3] = {0, 0, 0};
    for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
        const int d[3] = {dx, dy, dz};
        bool skip = (dx == 0 && dy == 0 && dz == 0);
        for (int a = 0; a < 3; ++a) if (grid[a] == 1 && d[a] != 0) skip = true;
        if (skip) continue;
        int q[3]; for (int a = 0; a < 3; ++a) q[a] = pmod(c0[a] + d[a], grid[a]);
        if (rid(q) != 0) peers.insert(rid(q));
    }
    printf("%ld %ld %d %d\n", checked, bad, shift_msgs, (int)peers.size());
    return 0;
}
'''


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    d = tmp_path_factory.mktemp("route")
    src = d / "route_driver.cpp"
    src.write_text(DRIVER)
    exe = d / "route_driver"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), "-o", str(exe)], check=True)
    return str(exe)


@pytest.mark.parametrize("grid,msgs", [((3, 3, 3), (6, 26)), ((2, 2, 2), (3, 7)), ((2, 2, 1), (2, 3)),
                                       ((2, 1, 1), (1, 1)), ((4, 3, 2), (5, 17)), ((1, 2, 2), (2, 3))])
def test_shift_equals_direct_and_message_counts(driver, grid, msgs):
    out = subprocess.run([driver, *map(str, grid)], check=True, capture_output=True, text=True).stdout.split()
    checked, bad, shift_msgs, direct_peers = map(int, out)
    assert checked > 50000 and bad == 0, (checked, bad)
    assert (shift_msgs, direct_peers) == msgs
