"""Host-side helpers of the multi-GPU spatial decomposition (C5): rank grid, block
extraction / reassembly of canonical lattices, and the NCCL-id bootstrap over torch.distributed.
Pure index bookkeeping (no method arithmetic); the exchange itself runs in libakmc.so (akmc_dist.cuh)."""
from __future__ import annotations

import numpy as np


def grid_for(world: int) -> tuple:
    """gpu_grid for 1/2/4/8 ranks: 1x1x1, 2x1x1, 2x2x1, 2x2x2."""
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(world) or (world, 1, 1)


def rank_coords(rank: int, grid) -> tuple:
    gx, gy, _ = grid
    return rank % gx, (rank // gx) % gy, rank // (gx * gy)


def _as_cells(species: np.ndarray, cells) -> np.ndarray:
    """canonical [2*(x + Lx*(y + Ly*z)) + b] -> array [z][y][x][b]"""
    Lx, Ly, Lz = cells
    return species.reshape(Lz, Ly, Lx, 2)


def block_of(global_species: np.ndarray, block_cells, grid, rank: int) -> np.ndarray:
    """This rank's block of a global canonical lattice, as a canonical block lattice."""
    bx, by, bz = block_cells
    G = (bx * grid[0], by * grid[1], bz * grid[2])
    cx, cy, cz = rank_coords(rank, grid)
    g = _as_cells(global_species, G)
    return np.ascontiguousarray(g[cz * bz:(cz + 1) * bz, cy * by:(cy + 1) * by, cx * bx:(cx + 1) * bx, :]).reshape(-1)


def assemble(blocks, block_cells, grid) -> np.ndarray:
    """Inverse of block_of over all ranks (blocks[r] canonical per rank)."""
    bx, by, bz = block_cells
    G = (bx * grid[0], by * grid[1], bz * grid[2])
    out = np.empty((G[2], G[1], G[0], 2), dtype=np.uint8)
    for r, blk in enumerate(blocks):
        cx, cy, cz = rank_coords(r, grid)
        out[cz * bz:(cz + 1) * bz, cy * by:(cy + 1) * by, cx * bx:(cx + 1) * bx, :] = blk.reshape(bz, by, bx, 2)
    return out.reshape(-1)


def broadcast_nccl_id(rank: int, device=None) -> bytes:
    """Rank 0 creates an ncclUniqueId through the C-ABI; torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist

    from .akmc import nccl_unique_id
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0)
    return bytes(buf.cpu().numpy().tobytes())
