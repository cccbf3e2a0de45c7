"""Multi-GPU monodomain step: slab partition, halo exchange, distributed PCG.

SURVEY.md §8(e). One process per GPU (torchrun), `torch.distributed` for the
plumbing (NCCL on GPUs; gloo in the CPU tests).  The path shards by nodes:
the ionic update, the RHS nodal terms and the activation map are node-local;
the operator needs a one-node halo and the CG needs global dot products.

Partition: the structured lattice is cut into contiguous slabs of z-planes
(the slowest lattice axis, so every rank's nodes - and each halo plane - are
contiguous in the reference's node numbering and go to NCCL without
packing).  A rank stores its owned planes plus one ghost plane per neighbour.

Per step: ionic update on owned nodes -> halo(combo, I^v, x0) -> PCG.
Per pipelined-PCG iteration (`mdx_pcg_phase`, csrc/solver.cu): halo(m) ->
sweep over owned rows -> one all-reduce of 4 partial sums -> host-side
alpha/beta/convergence (the same formulas as the single-GPU kernel).

`PipelinedPcgDriver` and `DistributedTissueSolver.step` are the host logic;
the device work goes through the hooks `_ionic`, `_prepare_solve` and
`phase` (sm_100a kernels).  tests/test_distributed.py runs the same host
logic over gloo with world size 2 and a CPU implementation of the hooks,
against the single-domain oracle.
"""

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NonFiniteSolution, SolverDivergence

PH_INIT, PH_W0, PH_SWEEP, PH_ZERO, PH_ACT = 0, 1, 2, 3, 4


# ---------------------------------------------------------------------------
# Partition
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class LocalSlab:
    rank: int
    nranks: int
    plane: int          # nodes per z-plane
    nz1: int            # planes of the global lattice
    k0: int             # owned planes [k0, k1)
    k1: int
    kl0: int            # stored planes [kl0, kl1) = owned + ghosts
    kl1: int

    @property
    def n_local(self):
        return (self.kl1 - self.kl0) * self.plane

    @property
    def global_begin(self):
        return self.kl0 * self.plane

    @property
    def own_begin(self):       # local row range of the owned nodes
        return (self.k0 - self.kl0) * self.plane

    @property
    def own_end(self):
        return (self.k1 - self.kl0) * self.plane

    @property
    def owned_global(self):
        return np.arange(self.k0 * self.plane, self.k1 * self.plane)

    def halo_plan(self):
        """[(peer, send_local_range, recv_local_range)] for this rank."""
        plan = []
        P = self.plane
        if self.k0 > 0:
            plan.append((self.rank - 1, (self.own_begin, self.own_begin + P), (0, P)))
        if self.k1 < self.nz1:
            e = self.own_end
            plan.append((self.rank + 1, (e - P, e), (e, e + P)))
        return plan


    def sweep_split(self):
        """((i0, i1), [boundary ranges]) of the owned local rows, or None.

        Interior rows have no ghost-plane neighbour (the 27-point row of a
        node in plane k reads planes k-1..k+1), so their CG sweep can run
        while the halo exchange of m is in flight; the boundary planes next to
        a ghost plane run after it lands.  None: no halo, or no interior."""
        P = self.plane
        lo = P if self.k0 > 0 else 0
        hi = P if self.k1 < self.nz1 else 0
        if not (lo or hi):
            return None
        i0, i1 = self.own_begin + lo, self.own_end - hi
        if i1 <= i0:
            return None
        bnd = []
        if lo:
            bnd.append((self.own_begin, i0))
        if hi:
            bnd.append((i1, self.own_end))
        return (i0, i1), bnd


def slab_partition(lattice, nranks):
    """Split the node planes of an (nx, ny, nz)-cell lattice into nranks slabs
    of near-equal plane counts (z-planes, contiguous in node numbering)."""
    nx, ny, nz = lattice
    nz1 = nz + 1
    if nranks > nz1:
        raise ValueError(f"{nranks} ranks exceed the {nz1} lattice planes")
    cuts = np.linspace(0, nz1, nranks + 1).round().astype(int)
    plane = (nx + 1) * (ny + 1)
    out = []
    for r in range(nranks):
        k0, k1 = int(cuts[r]), int(cuts[r + 1])
        out.append(LocalSlab(r, nranks, plane, nz1, k0, k1, max(k0 - 1, 0),
                             min(k1 + 1, nz1)))
    return out


# ---------------------------------------------------------------------------
# Communication (torch.distributed: NCCL on GPUs, gloo on CPU)
# ---------------------------------------------------------------------------


class SlabComm:
    def __init__(self, slab, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.slab = slab
        self.group = group
        self.plan = slab.halo_plan()
        self.single = dist.get_world_size(group) == 1

    def halo(self, *vectors):
        """Fill the ghost planes of each 1-D local vector from the neighbours."""
        self.halo_finish(self.halo_start(*vectors))

    def halo_start(self, *vectors):
        """Post the halo sends/receives; returns the pending exchange.

        NCCL moves device slices directly and its work runs on NCCL's stream
        (ordered after the work already enqueued on the current stream), so
        kernels enqueued before halo_finish overlap the transfer.  gloo (CPU
        tests, or several ranks sharing one GPU in the GPU tests) stages device
        slices through host copies."""
        if not self.plan:
            return None
        dist = self.dist
        staged = (dist.get_backend(self.group) == "gloo"
                  and any(v.is_cuda for v in vectors))
        ops, back = [], []
        for vec in vectors:
            for peer, (s0, s1), (r0, r1) in self.plan:
                snd, rcv = vec[s0:s1], vec[r0:r1]
                if staged:
                    snd = snd.cpu()
                    host = rcv.cpu()
                    back.append((rcv, host))
                    rcv = host
                ops.append(dist.P2POp(dist.isend, snd, peer, group=self.group))
                ops.append(dist.P2POp(dist.irecv, rcv, peer, group=self.group))
        return dist.batch_isend_irecv(ops), back

    def halo_finish(self, pending):
        """Complete a halo_start: NCCL makes the current stream wait for the
        transfer (no host block); gloo waits on the host and copies staged
        receives back to the device."""
        if pending is None:
            return
        reqs, back = pending
        for req in reqs:
            req.wait()
        for dev, host in back:
            dev.copy_(host)

    def allreduce(self, t):
        """Sum a small tensor over ranks in place; returns it."""
        if self.single:
            return t
        if t.is_cuda and self.dist.get_backend(self.group) == "gloo":
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return t
        self.dist.all_reduce(t, group=self.group)
        return t


# ---------------------------------------------------------------------------
# Backend-agnostic pipelined PCG driver
# ---------------------------------------------------------------------------


def _sweep_split(be):
    """The backend's interior/boundary row split for halo overlap, or None
    (no neighbours, no interior, or MDX_DIST_OVERLAP=0)."""
    if os.environ.get("MDX_DIST_OVERLAP", "1") == "0":
        return None
    sp = be.slab.sweep_split()
    if sp is None:
        return None
    # the split costs two more launches per boundary plane and iteration (a
    # host-enqueue cost): only worth it when the interior sweep is long enough
    # to hide the exchange - at least MDX_DIST_OVERLAP_MIN (default 4) times
    # the boundary rows
    ratio = float(os.environ.get("MDX_DIST_OVERLAP_MIN", "4"))
    (i0, i1), bnd = sp
    if i1 - i0 < ratio * sum(b1 - b0 for b0, b1 in bnd):
        return None
    return sp


class PipelinedPcgDriver:
    """Distributed pipelined Jacobi PCG (Ghysels-Vanroose), host side.

    backend must provide:
      phase(kind, alpha=0, beta=0, first=0, mbuf=0) -> local 4-vector tensor
      vectors: attributes x, combo, z, m(buf) and lift currents for halos
    The returned local sums are all-reduced here, so every rank computes the
    same alpha/beta and the same stopping decision.
    """

    def __init__(self, comm, backend, tol, max_iter):
        self.comm = comm
        self.be = backend
        self.tol = float(tol)
        self.max_iter = int(max_iter)

    def _sums(self, local):
        return self.comm.allreduce(local).cpu().numpy().astype(np.float64)

    def solve(self, tissue=True):
        be, comm = self.be, self.comm
        if tissue:
            comm.halo(be.x, be.combo, *be.lift_currents())
        else:
            comm.halo(be.x)
        s = self._sums(be.phase(PH_INIT))
        b_norm = math.sqrt(s[0])
        res = math.sqrt(s[1])
        rz = s[2]
        nonfinite = s[3]
        if b_norm == 0.0:
            be.phase(PH_ZERO)
            return 0, 0.0, False
        if res <= self.tol * b_norm:
            return 0, res / b_norm, nonfinite != 0.0
        comm.halo(be.z)
        s = self._sums(be.phase(PH_W0, mbuf=1))
        gamma, delta, gamma_prev, alpha_prev = rz, s[0], 0.0, 1.0
        for it in range(1, self.max_iter + 1):
            first = it == 1
            if first:
                beta, alpha = 0.0, gamma / delta
            else:
                beta = gamma / gamma_prev
                alpha = gamma / (delta - beta * gamma / alpha_prev)
            mbuf = (it - 1) & 1
            split = _sweep_split(be)
            if split is None:
                comm.halo(be.m_buffer(mbuf))
                local = be.phase(PH_SWEEP, alpha, beta, int(first), mbuf)
            else:
                # interior rows while the halo of m is in flight, then the
                # planes next to the ghosts; local sums in a fixed order
                pend = comm.halo_start(be.m_buffer(mbuf))
                local = be.phase(PH_SWEEP, alpha, beta, int(first), mbuf, rows=split[0])
                comm.halo_finish(pend)
                for rows in split[1]:
                    local = local + be.phase(PH_SWEEP, alpha, beta, int(first), mbuf,
                                             rows=rows)
            s = self._sums(local)
            nonfinite = s[3]
            res = math.sqrt(s[2])
            if res <= self.tol * b_norm:
                return it, res / b_norm, nonfinite != 0.0
            gamma_prev, alpha_prev, gamma, delta = gamma, alpha, s[0], s[1]
        return -self.max_iter, res / b_norm, nonfinite != 0.0


class DevicePcgDriver:
    """The same pipelined PCG with the scalar recurrences on the device.

    Every phase, all-reduce, halo exchange and scalar update is enqueued on
    the stream without reading anything back (NCCL collectives are
    stream-ordered); the host reads the 88-byte scalar state only after a
    chunk of iterations.  Phases enqueued after convergence are no-ops on the
    device (they gate on the state), so the iterate is exactly the one the
    host driver returns.  The first chunk is the previous solve's iteration
    count, then chunks of two.

    backend must provide phase_dev(kind, mbuf), scalars(phase) and
    read_scalars(), plus the vectors PipelinedPcgDriver uses.
    """

    def __init__(self, comm, backend, tol, max_iter, predict=8):
        self.comm = comm
        self.be = backend
        self.tol = float(tol)
        self.max_iter = int(max_iter)
        self.predict = max(1, int(predict))

    def solve(self, tissue=True):
        be, comm = self.be, self.comm
        if tissue:
            comm.halo(be.x, be.combo, *be.lift_currents())
        else:
            comm.halo(be.x)
        be.phase_dev(PH_INIT)
        comm.allreduce(be.sums)
        be.scalars(N.SC_INIT)
        be.phase_dev(PH_ZERO)
        comm.halo(be.z)
        be.phase_dev(PH_W0, mbuf=1)
        comm.allreduce(be.sums)
        be.scalars(N.SC_W0)
        it, chunk = 0, self.predict
        sc = None
        split = _sweep_split(be)
        while it < self.max_iter:
            for _ in range(min(chunk, self.max_iter - it)):
                it += 1
                mbuf = (it - 1) & 1
                if split is None:
                    comm.halo(be.m_buffer(mbuf))
                    be.phase_dev(PH_SWEEP, mbuf=mbuf)
                else:
                    # interior rows overlap the halo exchange of m
                    pend = comm.halo_start(be.m_buffer(mbuf))
                    be.phase_dev(PH_SWEEP, mbuf=mbuf, rows=split[0], part=0)
                    comm.halo_finish(pend)
                    for j, rows in enumerate(split[1]):
                        be.phase_dev(PH_SWEEP, mbuf=mbuf, rows=rows, part=j + 1)
                    be.combine_parts(1 + len(split[1]))
                comm.allreduce(be.sums)
                be.scalars(N.SC_SWEEP)
            sc = be.read_scalars()
            if sc.state != 0:
                break
            chunk = 2
        if sc is None:
            sc = be.read_scalars()
        if sc.state == 2:
            return 0, 0.0, False
        rel = sc.res / sc.b_norm
        if sc.state == 1:
            return sc.it, rel, sc.nonfinite != 0.0
        return -self.max_iter, rel, sc.nonfinite != 0.0


# ---------------------------------------------------------------------------
# GPU backend + tissue solver
# ---------------------------------------------------------------------------


class DistributedTissueSolver:
    """Monodomain time loop over `nranks` GPUs (one per process).

    Single-volume structured slabs (configs 0/2 and the reference benchmark
    slab).  The global operator tables are built once per rank on its GPU;
    each rank keeps only its slab of the vectors and ionic states.
    """

    def __init__(self, config, group=None, device_scalars=True):
        import torch
        import torch.distributed as dist

        from .fem import detect_lattice
        from .simulation import RING_SLOTS, TissueSolver

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.device_scalars = bool(device_scalars)
        self.launches = 0          # libmdx kernels enqueued (bench.py's gpu_launches)
        lattice = detect_lattice(config.mesh)
        if lattice is None:
            raise ValueError("the distributed solver needs a structured hex slab")
        if len([v for v in config.volumes if not v.disabled]) != 1:
            raise ValueError("the distributed solver supports one conducting volume")
        self.slab = slab_partition(lattice, self.nranks)[self.rank]
        self.comm = SlabComm(self.slab, group)
        # global setup (operators, initial state) on this rank's GPU, then keep
        # only the slab
        g = TissueSolver(config, operator="stencil")
        self.config = config
        self.n_global = g.n
        self.dt = g.dt
        self.step_index, self.time = 0, 0.0
        sl = self.slab
        gb, nl = sl.global_begin, sl.n_local
        lo, hi = gb, gb + nl
        f64 = dict(dtype=torch.float64, device="cuda")
        self.op = g.op
        self.meta = g.op.meta[lo:hi].contiguous()
        self.u_ring = torch.zeros((RING_SLOTS, nl), **f64)
        self.u_ring[:, :] = g.u_ring[:, lo:hi]
        self.head = 0
        vol = g.lift_volumes[0]
        own = np.arange(sl.own_begin, sl.own_end)
        own_glob = own + gb
        pos = np.searchsorted(vol.dofs, own_glob)
        if not np.array_equal(vol.dofs[np.minimum(pos, vol.dofs.size - 1)], own_glob):
            raise ValueError("the volume must cover every node")
        self.model_id = vol.module.MODEL_ID
        self.packed = vol.packed
        self.nv = vol.num_vars
        self.n_own = own.size
        self.w_ring = vol.w_ring[:, :, pos].contiguous()  # (slots, nv, n_own)
        self.dofs = torch.from_numpy(own.astype(np.int32)).cuda()
        self.currents = torch.zeros(nl, **f64)
        self.combo = torch.zeros(nl, **f64)
        self.profiles = (g.profiles[:, lo:hi].contiguous() if g.profiles is not None
                         else None)
        self._impulses = g._impulses
        self.act_time = g.act_time[lo:hi].contiguous()
        self.best_slope = g.best_slope[lo:hi].contiguous()
        self.frozen = g.frozen[lo:hi].contiguous()
        self.clamps = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        from .linalg import CgWorkspace

        self.ws = CgWorkspace(nl)
        self.sums = torch.zeros(4, **f64)
        self.sum_parts = torch.zeros((3, 4), **f64)   # interior + two boundary planes
        # device-resident PcgScal (88 bytes) for DevicePcgDriver
        self.scal = torch.zeros(C.sizeof(N.PcgScal) // 8 + 1, **f64)
        self.tol = config.linear_solver.tolerance
        self.max_iter = config.linear_solver.max_iterations
        self.bdf_order = config.bdf_order
        self.iters = []
        self.x = None
        del g

    # -- backend protocol for PipelinedPcgDriver --------------------------------
    def lift_currents(self):
        return (self.currents,)

    def m_buffer(self, k):
        nl = self.slab.n_local
        return self.ws.m[k * nl:(k + 1) * nl]

    @property
    def z(self):
        return self.ws.z

    def _rows_args(self, rows):
        """The solve's kernel arguments, restricted to local rows [r0, r1)
        (one copy per range and step, reused by every iteration)."""
        a = self._args
        if rows is None:
            return a
        b = self._rows_cache.get(rows)
        if b is None:
            b = N.CgArgs.from_buffer_copy(a)
            b.row_begin, b.row_end = rows
            self._rows_cache[rows] = b
        return b

    def phase(self, kind, alpha=0.0, beta=0.0, first=0, mbuf=0, rows=None):
        a = self._rows_args(rows)
        N.check(N.lib().mdx_pcg_phase(N.C.byref(a), kind, 1, alpha, beta, first, mbuf,
                                      N.ptr(self.sums), N.stream_handle()), "mdx_pcg_phase")
        self.launches += 2          # phase kernel + partial reduction
        return self.sums.clone()

    def phase_dev(self, kind, mbuf=0, rows=None, part=None):
        """part j: the local sums go to sum_parts[j] (combine_parts adds them)."""
        out = self.sums if part is None else self.sum_parts[part]
        N.check(N.lib().mdx_pcg_phase_dev(N.C.byref(self._rows_args(rows)), kind, 1,
                                          N.ptr(self.scal), mbuf, N.ptr(out),
                                          N.stream_handle()), "mdx_pcg_phase_dev")
        self.launches += 2

    def combine_parts(self, k):
        """sums = sum_parts[0] + ... + sum_parts[k-1] (fixed order)."""
        import torch

        torch.sum(self.sum_parts[:k], 0, out=self.sums)

    def scalars(self, phase):
        N.check(N.lib().mdx_pcg_scalars(N.ptr(self.sums), N.ptr(self.scal), phase, self.tol,
                                        self.max_iter, N.stream_handle()), "mdx_pcg_scalars")
        self.launches += 1

    def read_scalars(self):
        raw = self.scal.cpu().numpy().tobytes()
        return N.PcgScal.from_buffer_copy(raw[:C.sizeof(N.PcgScal)])

    # -- stepping (host logic shared with the CPU test backend) -----------------
    def step(self):
        from .simulation import RING_SLOTS

        order = min(self.step_index + 1, self.bdf_order)
        t_next = self.time + self.dt
        mask = 0
        for k, (protocol, i) in enumerate(self._impulses):
            if protocol.window_active(i, t_next):
                mask |= 1 << k
        head, nslot = self.head, (self.head + 1) % RING_SLOTS
        self._ionic(order, t_next, head, nslot, mask)
        self._prepare_solve(order, t_next, head, nslot)
        if self.device_scalars:
            it, rel, nonfinite = DevicePcgDriver(
                self.comm, self, self.tol, self.max_iter,
                predict=self.iters[-1] if self.iters else 8).solve(tissue=True)
        else:
            it, rel, nonfinite = PipelinedPcgDriver(self.comm, self, self.tol,
                                                    self.max_iter).solve(tissue=True)
        if it < 0:
            raise SolverDivergence(-it, rel)
        if nonfinite:
            raise NonFiniteSolution("linear solve produced non-finite entries")
        if self.device_scalars:
            self.phase_dev(PH_ACT)
        else:
            self.phase(PH_ACT)
        self.iters.append(it)
        self.head = nslot
        self.step_index += 1
        self.time = t_next
        return it

    def potential_local(self):
        return self.u_ring[self.head]

    # -- device hooks -----------------------------------------------------------
    def _ionic(self, order, t_next, head, nslot, mask):
        from .simulation import RING_SLOTS

        sl = self.slab
        ia = N.TissueIonicArgs(
            n=self.n_own, dofs=N.ptr(self.dofs), u_ring=N.ptr(self.u_ring),
            ldu=sl.n_local, w_ring=N.ptr(self.w_ring), ldw=self.n_own,
            ring_slots=RING_SLOTS, head=head, order=order, prep=1, dt=self.dt,
            i_out=N.ptr(self.currents), clamp_count=N.ptr(self.clamps),
            combo=N.ptr(self.combo), profiles=N.ptr(self.profiles), ldp=sl.n_local,
            active_mask=mask, n_impulses=len(self._impulses), status=N.ptr(self.status))
        Ph, Pp = N.host_doubles(self.packed)
        N.check(N.lib().mdx_tissue_ionic(self.model_id, N.C.byref(ia), Pp, int(Ph.size),
                                         N.stream_handle()), "mdx_tissue_ionic")
        self.launches += 1

    def _prepare_solve(self, order, t_next, head, nslot):
        sl = self.slab
        self.x = self.u_ring[nslot]
        a = N.CgArgs()
        op = self.op
        a.op = op.operator()
        a.op.n = sl.n_local
        a.op.nz1 = sl.kl1 - sl.kl0
        a.op.meta = N.ptr(self.meta)
        a.a_val = N.ptr(op.a_tables[order])
        a.dinv = N.ptr(op.dinv[order])
        a.m_val = N.ptr(op.d_m)
        a.combo = N.ptr(self.combo)
        a.n_lift = 1
        a.lift_val[0] = N.ptr(op.d_lift[0])
        a.lift_cur[0] = N.ptr(self.currents)
        a.inactive = N.ptr(op.d_inactive)
        a.rest = N.ptr(op.d_rest)
        a.thr = N.ptr(op.d_thr)
        a.x = N.ptr(self.x)
        a.u_prev = N.ptr(self.u_ring[head])
        a.act_time = N.ptr(self.act_time)
        a.best_slope = N.ptr(self.best_slope)
        a.frozen = N.ptr(self.frozen)
        a.t_next = t_next
        a.dt = self.dt
        self.ws.fill(a)
        a.status = N.ptr(self.status)
        a.row_begin, a.row_end = sl.own_begin, sl.own_end
        self._args = a
        self._rows_cache = {}

    def gather_potential(self):
        """Full potential on every rank (all-gather of the owned slabs)."""
        import torch
        import torch.distributed as dist

        sl = self.slab
        slabs = slab_partition_from(sl)
        sizes = [(p.k1 - p.k0) * p.plane for p in slabs]
        width = max(sizes)          # equal-size messages (gloo requires it)
        own = self.potential_local()[sl.own_begin:sl.own_end]
        buf = torch.zeros(width, dtype=own.dtype, device=own.device)
        buf[:own.numel()] = own
        parts = [torch.empty_like(buf) for _ in slabs]
        dist.all_gather(parts, buf, group=self.comm.group)
        return torch.cat([p[:k] for p, k in zip(parts, sizes)]).cpu().numpy()


def slab_partition_from(sl):
    """All ranks' slabs from one rank's LocalSlab (same cut rule)."""
    cuts = np.linspace(0, sl.nz1, sl.nranks + 1).round().astype(int)
    return [LocalSlab(r, sl.nranks, sl.plane, sl.nz1, int(cuts[r]), int(cuts[r + 1]),
                      max(int(cuts[r]) - 1, 0), min(int(cuts[r + 1]) + 1, sl.nz1))
            for r in range(sl.nranks)]
