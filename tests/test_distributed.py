"""Multi-rank host logic of the distributed solver, on CPU over gloo.

The partition/halo/pipelined-PCG/step logic of
paper_2308_01651_b200.distributed runs in 2 (and 3) processes with the CPU
hook implementation of tests/dist_cpu.py; the gathered potential, CG
iteration counts and activation map must match the single-domain oracle
(which is pinned bit-for-bit to the reference).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2308_01651_b200.distributed import slab_partition


def test_slab_partition_covers_lattice_once():
    for lattice, nr in (((40, 14, 6), 2), ((40, 14, 6), 3), ((200, 70, 30), 8),
                        ((4, 4, 4), 5)):
        slabs = slab_partition(lattice, nr)
        plane = (lattice[0] + 1) * (lattice[1] + 1)
        owned = np.concatenate([s.owned_global for s in slabs])
        assert np.array_equal(owned, np.arange(plane * (lattice[2] + 1)))
        for s in slabs:
            assert s.k1 > s.k0
            assert s.n_local == (s.kl1 - s.kl0) * plane
            # every halo send range is owned, every recv range is a ghost plane
            for peer, (a0, a1), (b0, b1) in s.halo_plan():
                assert s.own_begin <= a0 < a1 <= s.own_end
                assert b1 <= s.own_begin or b0 >= s.own_end
                assert a1 - a0 == b1 - b0 == plane
                other = slabs[peer]
                assert any(p == s.rank for p, _, _ in other.halo_plan())
    with pytest.raises(ValueError):
        slab_partition((4, 4, 2), 4)


def test_sweep_split_rows():
    """Interior rows never read a ghost plane; interior + boundary = owned."""
    for lattice, nr in (((40, 14, 6), 2), ((40, 14, 6), 3), ((200, 70, 30), 8),
                        ((4, 4, 3), 4), ((4, 4, 4), 1)):
        plane = (lattice[0] + 1) * (lattice[1] + 1)
        for s in slab_partition(lattice, nr):
            sp = s.sweep_split()
            ghosts = [(r0, r1) for _, _, (r0, r1) in s.halo_plan()]
            if sp is None:
                assert not ghosts or s.k1 - s.k0 <= len(ghosts)
                continue
            (i0, i1), bnd = sp
            rows = sorted([(i0, i1)] + bnd)
            assert rows[0][0] == s.own_begin and rows[-1][1] == s.own_end
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            # the interior's stencil reach (one plane either side) misses the ghosts
            for g0, g1 in ghosts:
                assert i1 + plane <= g0 or i0 - plane >= g1
            assert len(bnd) == len(ghosts)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, steps, out_dir, device_scalars=False):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["MDX_DIST_OVERLAP_MIN"] = "0"     # exercise the split on the small slab
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu import CpuSlabTissue
        from paper_2308_01651_b200 import configs

        cfg = configs.config0(configs.this_package(), h=1e-3)
        solver = CpuSlabTissue(cfg, device_scalars=device_scalars)
        for _ in range(steps):
            solver.step()
        u = solver.gather_potential()
        sl = solver.slab
        act = solver.act.copy()
        frozen = solver.frozen.copy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u,
                 iters=np.array(solver.iters),
                 act=act[sl.own_begin:sl.own_end],
                 frozen=frozen[sl.own_begin:sl.own_end],
                 split_rows=np.array(sorted(solver.sweep_rows_seen)).reshape(-1, 2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,device_scalars", [(2, False), (3, False), (2, True), (3, True)])
def test_distributed_step_matches_single_domain_oracle(tmp_path, world, device_scalars):
    """Host-driven (PipelinedPcgDriver) and device-scalar (DevicePcgDriver:
    chunked enqueue, phases gated on the scalar state) distributed steps."""
    from oracle import monodomain_oracle as O
    from paper_2308_01651_b200 import configs

    steps = 60
    mp.spawn(_worker, args=(world, _free_port(), steps, str(tmp_path), device_scalars),
             nprocs=world, join=True)
    cfg = configs.config0(configs.this_package(), h=1e-3)
    orc = O.OracleTissue(cfg)
    for _ in range(steps):
        orc.step()
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in res:
        np.testing.assert_array_equal(r["u"], res[0]["u"])           # all ranks agree
        np.testing.assert_array_equal(r["iters"], res[0]["iters"])
    if world == 2:
        # every rank swept its interior plane during the halo exchange and its
        # plane next to the ghost after it (distributed.py sweep overlap)
        for r in res:
            assert len(r["split_rows"]) == 2, r["split_rows"]
    its = res[0]["iters"]
    assert np.abs(its - np.array(orc.iters)).max() <= 1
    u = res[0]["u"]
    rel = np.linalg.norm(u - orc.potential) / np.linalg.norm(orc.potential)
    assert rel < 1e-9, rel
    act = np.concatenate([r["act"] for r in res])
    frozen = np.concatenate([r["frozen"] for r in res]).astype(bool)
    amap = np.where(frozen, act, -1.0)
    ref = orc.activation_map
    assert np.array_equal(amap >= 0, ref >= 0)
    both = (amap >= 0) & (ref >= 0)
    assert np.abs(amap[both] - ref[both]).max() <= cfg.dt * (1 + 1e-9)
