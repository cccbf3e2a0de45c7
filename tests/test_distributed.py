"""Multi-rank host logic of the distributed solver, on CPU over gloo.

The RCB partition, rank-local problems, halo plans/exchange and the
pipelined-PCG drivers of paper_2308_01651_b200.distributed run in 2 and 3
processes with the CPU hooks of tests/dist_cpu.py; the gathered potential,
CG iteration counts and activation map must match the single-domain oracle
(pinned bit-for-bit to the reference) on configs 0, 3 and 4 (reduced sizes).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2308_01651_b200.partition import (build_part, grid_coords, grid_of, halo_plans,
                                             partition, rcb, send_lists)


def _cfg(name):
    from paper_2308_01651_b200 import configs, ventricle

    ns = configs.this_package()
    if name == "cfg0":
        return configs.config0(ns, h=1e-3)
    if name == "cfg3":
        return configs.config3(ns, h=1e-3, seed=7)
    if name == "cfg4":
        return ventricle.config4(ns, n_xi=3, n_th=12, n_ph=32)
    raise KeyError(name)


def test_rcb_balanced_deterministic():
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((1000, 3)) * (5.0, 1.0, 0.2)
    for k in (1, 2, 3, 5, 8):
        p = rcb(pts, k)
        sizes = np.bincount(p, minlength=k)
        assert sizes.sum() == 1000 and sizes.min() >= 1000 // k - 1
        assert sizes.max() <= -(-1000 // k) + 1
        np.testing.assert_array_equal(p, rcb(pts, k))
    # the first cut is across the longest axis
    p = rcb(pts, 2)
    assert pts[p == 0, 0].max() <= pts[p == 1, 0].min()
    with pytest.raises(ValueError):
        rcb(pts[:3], 4)


@pytest.mark.parametrize("name", ["cfg0", "cfg3", "cfg4"])
@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_local_problems(name, nranks):
    """Every owned node's element star is local; send/recv lists agree
    between ranks; on logical grids every part is a box whose local operator
    pattern compresses to the same diagonals as the global one."""
    import torch

    from paper_2308_01651_b200.fem import FeSpace
    from paper_2308_01651_b200.operators import DiaOperator

    mesh = _cfg(name).mesh
    owner = partition(mesh, nranks)
    assert np.bincount(owner).min() > 0
    g = grid_of(mesh)
    assert g is not None
    parts = halo_plans(mesh, owner)
    el = mesh.elements
    n_glob_pat = FeSpace(mesh).pattern()
    glob_plan = DiaOperator.plan(torch.from_numpy(n_glob_pat[0]),
                                 torch.from_numpy(n_glob_pat[1]), mesh.num_nodes)
    for p in parts:
        own = np.flatnonzero(owner == p.rank)
        np.testing.assert_array_equal(np.sort(p.nodes[p.owned]), own)
        star = np.flatnonzero(np.isin(el, own).any(axis=1))
        assert np.isin(star, p.elements).all()
        assert np.all(np.diff(p.elements) > 0)              # ascending global order
        np.testing.assert_array_equal(mesh.elements[p.elements], p.nodes[p.conn])
        # a part is a logical box: its owned coordinates span a product range
        c = grid_coords(g[0], own)
        span = np.prod([np.unique(c[:, a]).size for a in range(3)])
        assert span == own.size
        # the product's communication-free send lists equal the plan's
        sl = send_lists(mesh, owner, p)
        assert sorted(sl) == sorted(p.send)
        for q in sl:
            np.testing.assert_array_equal(sl[q], p.send[q])
            other = parts[q]
            np.testing.assert_array_equal(p.nodes[p.send[q]], other.nodes[other.recv[p.rank]])
        # local pattern: diagonal structure kept
        from paper_2308_01651_b200.geometry import Mesh

        loc = Mesh(mesh.nodes[p.nodes], p.conn, mesh.element_kind, mesh.material_ids[p.elements])
        ip, ix = FeSpace(loc).pattern()
        plan = DiaOperator.plan(torch.from_numpy(ip), torch.from_numpy(ix), loc.num_nodes)
        assert plan is not None and len(plan["pos"]) <= len(glob_plan["pos"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, steps, out_dir, device_scalars):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["OMP_NUM_THREADS"] = "1"
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu import CpuPartTissue

        solver = CpuPartTissue(_cfg(name), device_scalars=device_scalars)
        for _ in range(steps):
            solver.step()
        u = solver.gather_potential()
        amap = solver.gather_activation_map()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u, act=amap,
                 iters=np.array(solver.iters), sel=np.array(sorted(solver.sel_seen)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,device_scalars,steps", [
    ("cfg0", 2, False, 60), ("cfg0", 3, True, 60),
    ("cfg3", 2, True, 40), ("cfg3", 3, False, 40),
    ("cfg4", 2, True, 40), ("cfg4", 3, True, 40)])
def test_distributed_step_matches_single_domain_oracle(tmp_path, name, world, device_scalars,
                                                       steps):
    """Host-driven (PipelinedPcgDriver) and device-scalar (DevicePcgDriver)
    distributed steps against the single-domain oracle."""
    from oracle import monodomain_oracle as O

    mp.spawn(_worker, args=(world, _free_port(), name, steps, str(tmp_path), device_scalars),
             nprocs=world, join=True)
    cfg = _cfg(name)
    orc = O.OracleTissue(cfg)
    for _ in range(steps):
        orc.step()
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in res:
        np.testing.assert_array_equal(r["u"], res[0]["u"])           # all ranks agree
        np.testing.assert_array_equal(r["iters"], res[0]["iters"])
        # interior rows swept during the halo exchange, boundary rows after it
        assert set(r["sel"].tolist()) == {1, 2}, r["sel"]
    its = res[0]["iters"]
    assert np.abs(its - np.array(orc.iters)).max() <= 1
    u = res[0]["u"]
    rel = np.linalg.norm(u - orc.potential) / np.linalg.norm(orc.potential)
    assert rel < 1e-9, rel
    amap, ref = res[0]["act"], orc.activation_map
    assert np.array_equal(amap >= 0, ref >= 0)
    both = (amap >= 0) & (ref >= 0)
    if both.any():
        assert np.abs(amap[both] - ref[both]).max() <= cfg.dt * (1 + 1e-9)
