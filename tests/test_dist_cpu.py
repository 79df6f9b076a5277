"""Multi-process host-side checks of the spatial decomposition (gloo, world_size 2, CPU): block
extraction / reassembly of the global lattice and the rank grid used by the multi-GPU C5 path."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth
from paper_2604_24091_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid, block, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    G = tuple(b * g for b, g in zip(block, grid))
    glob = synth.make_lattice(G, 1, synth.fe_cu_fractions(0.1), 20, seed=9)
    blk = D.block_of(glob, block, grid, rank)
    parts = [None] * world
    tdist.all_gather_object(parts, blk)
    ok = np.array_equal(D.assemble(parts, block, grid), glob)
    # vacancies of each block map back to the global vacancy set (global slot ids = rank of site)
    vs = []
    for r, b in enumerate(parts):
        cx, cy, cz = D.rank_coords(r, grid)
        for i in np.flatnonzero(b == 6):
            bb = i & 1; c = i >> 1
            x, y, z = c % block[0], (c // block[0]) % block[1], c // (block[0] * block[1])
            gx, gy, gz = x + cx * block[0], y + cy * block[1], z + cz * block[2]
            vs.append(2 * (gx + G[0] * (gy + G[1] * gz)) + bb)
    ok &= np.array_equal(np.sort(vs), np.flatnonzero(glob == 6))
    q.put((rank, bool(ok)))
    tdist.destroy_process_group()


@pytest.mark.parametrize("grid", [(2, 1, 1), (1, 2, 1), (2, 2, 2)])
def test_block_decomposition_gloo(grid):
    world = grid[0] * grid[1] * grid[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, (8, 8, 8), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_grid_for():
    assert D.grid_for(1) == (1, 1, 1) and D.grid_for(8) == (2, 2, 2)
    for w in (1, 2, 4, 8):
        g = D.grid_for(w)
        assert g[0] * g[1] * g[2] == w
        assert sorted(D.rank_coords(r, g) for r in range(w)) == sorted(
            (x, y, z) for z in range(g[2]) for y in range(g[1]) for x in range(g[0]))
