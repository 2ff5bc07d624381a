"""Multi-rank brick decomposition on CPU (gloo, world sizes 2 and 4).

Each rank owns its brick's particles, builds the ghost layer through the
point-to-point exchange, and evaluates its forces with the oracle (owned x
owned + owned x ghosts); forces and the summed pair count must equal the
single-domain oracle's periodic result.  Migration and the planned
re-exchange are checked too."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import P, forces_close


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _state(n=2500, rho=0.5, seed=3):
    rng = np.random.default_rng(seed)
    L = (n / rho) ** (1 / 3)
    k = int(np.ceil(n ** (1 / 3)))
    grid = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), -1).reshape(-1, 3)[:n]
    pos = (grid + 0.5) * (L / k) + rng.uniform(-0.25, 0.25, (n, 3)) * (L / k)
    return np.mod(pos, L), L


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2512_03565_b200.decomposition import BrickDecomposition
        pos, L = _state()
        params = P(cutoff=2.5, skin=0.3)
        dec = BrickDecomposition(np.zeros(3), np.full(3, L), params.interaction_length, rank, world)
        ids = np.arange(len(pos), dtype=np.float64)
        allrows = torch.as_tensor(np.concatenate([pos, ids[:, None]], axis=1))
        # every rank starts with a scattered share, migration sorts it out
        share = allrows[rank::world].clone()
        owned = dec.migrate(share)
        assert bool((dec.owner_of(owned[:, :3]) == rank).all())
        n_tot = torch.tensor([owned.shape[0]])
        dist.all_reduce(n_tot)
        assert int(n_tot) == len(pos)
        ghosts = dec.plan(owned)
        op = owned[:, :3].numpy()
        gp = ghosts[:, :3].numpy()
        f1, _, s1 = O.pair_sweep(op, op, params, False, True, "one_by_v", 8)
        f2, _, s2 = O.pair_sweep(op, gp, params, False, False, "one_by_v", 8,
                                 own_j=np.ones(len(gp), dtype=np.int8))
        forces = f1 + f2
        ref_f, ref_st = O.force_phase_lc(pos, np.zeros(3), np.full(3, L), [True] * 3, params,
                                         "lc_c01", False, "one_by_v", 8)
        my_ids = owned[:, 3].numpy().astype(np.int64)
        ok = forces_close(forces, ref_f[my_ids])
        pairs = torch.tensor([s1.pair_interactions + s2.pair_interactions])
        dist.all_reduce(pairs)
        # re-exchange after small moves: same ghosts, moved with their owners
        rng = np.random.default_rng(100 + rank)
        moved = owned.clone()
        moved[:, :3] += torch.as_tensor(rng.uniform(-0.05, 0.05, (owned.shape[0], 3)))
        g2 = dec.exchange(moved)
        same_ids = bool(torch.equal(g2[:, 3], ghosts[:, 3]))
        disp = (g2[:, :3] - ghosts[:, :3]).abs().max().item() if len(g2) else 0.0
        with open(os.path.join(result_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(f"{int(ok)} {int(pairs)} {ref_st.pair_interactions} {int(same_ids)} {disp}\n")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bricks_match_single_domain(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok, pairs, ref_pairs, same_ids, disp = open(tmp_path / f"r{r}.txt").read().split()
        assert ok == "1", r
        assert int(pairs) == int(ref_pairs)
        assert same_ids == "1"
        assert float(disp) <= 0.05 + 1e-12


def test_brick_grid_and_geometry():
    from paper_2512_03565_b200.decomposition import BrickDecomposition, brick_grid
    assert brick_grid(1) == (1, 1, 1) and brick_grid(2) == (2, 1, 1)
    assert brick_grid(4) == (2, 2, 1) and brick_grid(8) == (2, 2, 2)
    d = BrickDecomposition(np.zeros(3), np.full(3, 20.0), 2.8, rank=5, nranks=8)
    assert d.coords == (1, 0, 1)
    assert d.brick_lo.tolist() == [10.0, 0.0, 10.0] and d.brick_hi.tolist() == [20.0, 10.0, 20.0]
    pos = torch.tensor([[10.0, 0.0, 10.0], [9.999, 9.999, 19.999], [-0.5, 20.5, 3.0]],
                       dtype=torch.float64)
    assert d.owner_of(pos).tolist() == [5, 4, 1]
    with pytest.raises(ValueError):
        BrickDecomposition(np.zeros(3), np.full(3, 10.0), 2.8, rank=0, nranks=2)
