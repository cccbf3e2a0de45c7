"""Multi-GPU monodomain step: RCB partition, halo exchange, distributed PCG.

SURVEY.md section 8(e).  One process per GPU (torchrun), `torch.distributed`
for the plumbing (NCCL on GPUs; gloo in the CPU tests).  The path shards by
nodes: the ionic update, the RHS nodal terms and the activation map are
node-local; the operator needs a one-node halo and the CG global dot
products.

Partition (partition.py): recursive coordinate bisection - of the logical
grid when the mesh has one (structured slabs, the config-4 ventricle: every
part is a box and its local operator keeps the global diagonal structure),
else of the node coordinates.  Each rank sets up ONLY its local problem: the
elements touching its nodes (ascending global order, so the owned rows are
the reference's rows bit for bit) and their nodes, as a local TissueSolver
(operators, ionic state stores of every volume, stimulus profiles,
activation map) built from a local SimulationConfig.

Per step: ionic update of the local volumes -> halo(x0, combo, I^v) ->
pipelined Jacobi PCG (Ghysels-Vanroose: one all-reduce of 4 sums and one
halo of m per iteration; `mdx_pcg_phase_dev`, scalar recurrences on the
device) -> activation.  The sweep of the owned rows next to a ghost runs
after the halo lands; the interior rows overlap the exchange (row classes
in `row_mask`, `mdx_cg_args.row_select`).  Halo packing is `mdx_gather` /
`mdx_scatter` into one contiguous buffer per direction; NCCL moves one slice
per peer.

`PipelinedPcgDriver` / `DevicePcgDriver` are the host logic (backend-
agnostic); tests/dist_cpu.py runs them, with the same partition and halo
code, over gloo with CPU hooks against the single-domain oracle.
"""

import ctypes as C
import dataclasses
import math
import os

import numpy as np

from . import _native as N
from .errors import NonFiniteSolution, SolverDivergence
from .partition import build_part, partition, send_lists

PH_INIT, PH_W0, PH_SWEEP, PH_ZERO, PH_ACT = 0, 1, 2, 3, 4
ROW_INTERIOR, ROW_BOUNDARY = 1, 2          # row_mask classes (0 = ghost)


# ---------------------------------------------------------------------------
# Local problem
# ---------------------------------------------------------------------------


def row_classes(part):
    """uint8 per local row: 1 owned interior, 2 owned next to a ghost (it is
    sent to a peer), 0 ghost."""
    cls = np.zeros(part.n_local, np.uint8)
    cls[part.owned] = ROW_INTERIOR
    for idx in part.send.values():
        cls[idx] = ROW_BOUNDARY
    return cls


def local_config(config, part):
    """The rank's SimulationConfig: local mesh (our types), fibers restricted
    to its nodes, the volumes present locally; everything else unchanged."""
    from .geometry import ElementKind, FiberField, Mesh
    from .simulation import SimulationConfig

    mesh = config.mesh
    kind = ElementKind(mesh.element_kind.value)
    mats = np.asarray(mesh.material_ids)[part.elements]
    loc = Mesh(np.asarray(mesh.nodes)[part.nodes], part.conn, kind, mats)
    fib = config.fibers
    fibers = FiberField(np.asarray(fib.f0)[part.nodes], np.asarray(fib.s0)[part.nodes],
                        np.asarray(fib.n0)[part.nodes])
    present = set(int(m) for m in np.unique(mats))
    vols = tuple(v for v in config.volumes if present & {int(m) for m in v.material_ids})
    fields = {f.name: getattr(config, f.name) for f in dataclasses.fields(SimulationConfig)
              if hasattr(config, f.name)}
    fields.update(mesh=loc, fibers=fibers, volumes=vols)
    return SimulationConfig(**fields)


# ---------------------------------------------------------------------------
# Communication (torch.distributed: NCCL on GPUs, gloo on CPU)
# ---------------------------------------------------------------------------


class HaloComm:
    """Ghost exchange of local vectors plus the small all-reduce."""

    def __init__(self, part, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.single = dist.get_world_size(group) == 1
        self.peers = sorted(set(part.send) | set(part.recv))
        dev = device if device is not None else "cpu"
        self.cuda = torch.device(dev).type == "cuda"
        self.send_idx, self.recv_idx = [], []
        self.send_off, self.recv_off = [0], [0]
        for q in self.peers:
            s = np.asarray(part.send.get(q, np.empty(0, np.int64)), np.int64)
            r = np.asarray(part.recv.get(q, np.empty(0, np.int64)), np.int64)
            self.send_idx.append(s)
            self.recv_idx.append(r)
            self.send_off.append(self.send_off[-1] + s.size)
            self.recv_off.append(self.recv_off[-1] + r.size)
        cat = lambda xs: np.concatenate(xs) if xs else np.empty(0, np.int64)  # noqa: E731
        self.d_send = torch.from_numpy(cat(self.send_idx)).to(dev)
        self.d_recv = torch.from_numpy(cat(self.recv_idx)).to(dev)
        self.nsend, self.nrecv = self.send_off[-1], self.recv_off[-1]
        self._bufs = {}
        self._ops = {}
        self.bytes_per_vector = 8 * (self.nsend + self.nrecv)

    def _buffers(self, k, like):
        import torch

        key = (k, like.device.type)
        if key not in self._bufs:
            self._bufs[key] = (torch.empty(k * max(self.nsend, 1), dtype=torch.float64,
                                           device=like.device),
                               torch.empty(k * max(self.nrecv, 1), dtype=torch.float64,
                                           device=like.device))
        return self._bufs[key]

    def _gather(self, vec, out):
        if self.nsend == 0:
            return
        if vec.is_cuda:
            N.check(N.lib().mdx_gather(self.nsend, N.ptr(self.d_send), N.ptr(vec), N.ptr(out),
                                       N.stream_handle()), "mdx_gather")
        else:
            out.copy_(vec[self.d_send])

    def _scatter(self, src, vec):
        if self.nrecv == 0:
            return
        if vec.is_cuda:
            N.check(N.lib().mdx_scatter(self.nrecv, N.ptr(self.d_recv), N.ptr(src), N.ptr(vec),
                                        N.stream_handle()), "mdx_scatter")
        else:
            vec[self.d_recv] = src

    def halo(self, *vectors):
        """Fill the ghost entries of each local vector from their owners."""
        self.halo_finish(self.halo_start(*vectors))

    def halo_start(self, *vectors):
        """Pack and post the exchange; returns the pending state.  NCCL runs
        the transfer on its own stream, ordered after the packing, so kernels
        enqueued before halo_finish overlap it.  gloo with device tensors (the
        GPU tests' shared-GPU ranks) stages through host copies."""
        if not self.peers or self.single:
            return None
        dist = self.dist
        k = len(vectors)
        sbuf, rbuf = self._buffers(k, vectors[0])
        for j, v in enumerate(vectors):
            self._gather(v, sbuf[j * self.nsend:(j + 1) * self.nsend])
        staged = dist.get_backend(self.group) == "gloo" and sbuf.is_cuda
        s_host = sbuf.cpu() if staged else sbuf
        r_host = rbuf.cpu() if staged else rbuf
        # the pack buffers persist, so the op list of a (count, device) pair is built
        # once (per CG iteration this is the host's largest cost on the exchange)
        key = (k, sbuf.device.type)
        ops = None if staged else self._ops.get(key)
        if ops is None:
            ops = []
            for i, q in enumerate(self.peers):
                for j in range(k):
                    s0, s1 = self.send_off[i], self.send_off[i + 1]
                    r0, r1 = self.recv_off[i], self.recv_off[i + 1]
                    if s1 > s0:
                        ops.append(dist.P2POp(dist.isend,
                                              s_host[j * self.nsend + s0:j * self.nsend + s1],
                                              q, group=self.group))
                    if r1 > r0:
                        ops.append(dist.P2POp(dist.irecv,
                                              r_host[j * self.nrecv + r0:j * self.nrecv + r1],
                                              q, group=self.group))
            if not staged:
                self._ops[key] = ops
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, vectors, rbuf, r_host if staged else None

    def halo_finish(self, pending):
        if pending is None:
            return
        reqs, vectors, rbuf, r_host = pending
        for req in reqs:
            req.wait()
        if r_host is not None:
            rbuf.copy_(r_host)
        for j, v in enumerate(vectors):
            self._scatter(rbuf[j * self.nrecv:(j + 1) * self.nrecv], v)

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
# Backend-agnostic pipelined PCG drivers
# ---------------------------------------------------------------------------


def _overlap(be):
    """Sweep the interior rows during the halo exchange of m, the boundary
    rows after it (MDX_DIST_OVERLAP=0: one sweep after the exchange)."""
    return (os.environ.get("MDX_DIST_OVERLAP", "1") != "0" and not be.comm.single
            and be.has_interior)


class PipelinedPcgDriver:
    """Distributed pipelined Jacobi PCG (Ghysels-Vanroose), host scalars.

    backend: phase(kind, alpha, beta, first, mbuf, sel) -> local 4 sums;
    vectors x, combo, z, m_buffer(k), lift_currents() for the halos.  The
    sums are all-reduced here, so every rank takes the same decisions.
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
        split = _overlap(be)
        for it in range(1, self.max_iter + 1):
            first = it == 1
            if first:
                beta, alpha = 0.0, gamma / delta
            else:
                beta = gamma / gamma_prev
                alpha = gamma / (delta - beta * gamma / alpha_prev)
            mbuf = (it - 1) & 1
            if not split:
                comm.halo(be.m_buffer(mbuf))
                local = be.phase(PH_SWEEP, alpha, beta, int(first), mbuf)
            else:
                pend = comm.halo_start(be.m_buffer(mbuf))
                local = be.phase(PH_SWEEP, alpha, beta, int(first), mbuf, sel=ROW_INTERIOR)
                comm.halo_finish(pend)
                local = local + be.phase(PH_SWEEP, alpha, beta, int(first), mbuf,
                                         sel=ROW_BOUNDARY)
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
    the stream without reading anything back (NCCL is stream-ordered); the
    host reads the 88-byte scalar state only after a chunk of iterations.
    Phases enqueued after convergence are no-ops on the device (they gate on
    the state), so the iterate is exactly the host driver's.  The first chunk
    is the previous solve's iteration count minus one, then chunks of two.

    backend: phase_dev(kind, mbuf, sel, part), combine_parts(k),
    scalars(phase), read_scalars(), `sums`, plus PipelinedPcgDriver's vectors.
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
        split = _overlap(be)
        while it < self.max_iter:
            for _ in range(min(chunk, self.max_iter - it)):
                it += 1
                mbuf = (it - 1) & 1
                if not split:
                    comm.halo(be.m_buffer(mbuf))
                    be.phase_dev(PH_SWEEP, mbuf=mbuf)
                else:
                    pend = comm.halo_start(be.m_buffer(mbuf))
                    be.phase_dev(PH_SWEEP, mbuf=mbuf, sel=ROW_INTERIOR, part=0)
                    comm.halo_finish(pend)
                    be.phase_dev(PH_SWEEP, mbuf=mbuf, sel=ROW_BOUNDARY, part=1)
                    be.combine_parts(2)
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
# GPU solver
# ---------------------------------------------------------------------------


class DistributedTissueSolver:
    """Monodomain time loop over `nranks` GPUs (one per process).

    Any mesh and any number of volumes (configs 0-4).  Each rank builds its
    own local problem only (partition.py) and a local TissueSolver for it;
    the step runs the local ionic launches, then the distributed pipelined
    PCG over the owned rows.
    """

    def __init__(self, config, group=None, operator="auto", owner=None, gate_scheme="bdf"):
        import torch
        import torch.distributed as dist

        from .simulation import TissueSolver

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.launches = 0
        mesh = config.mesh
        self.owner = partition(mesh, self.nranks) if owner is None else np.asarray(owner)
        part = build_part(mesh, self.owner, self.rank)
        part.send = send_lists(mesh, self.owner, part)
        self.part = part
        self.n_global = mesh.nodes.shape[0]
        self.config = config
        self.local = TissueSolver(local_config(config, part), operator=operator, cg_variant=2,
                                  gate_scheme=gate_scheme)
        loc = self.local
        self.n_local = loc.n
        self.comm = HaloComm(part, group, device="cuda")
        cls = row_classes(part)
        self.has_interior = bool((cls == ROW_INTERIOR).any())
        self.row_mask = torch.from_numpy(cls).cuda()
        self.owned_idx = torch.from_numpy(part.owned_local()).cuda()
        self.owned_global = torch.from_numpy(part.nodes[part.owned_local()]).cuda()
        f64 = dict(dtype=torch.float64, device="cuda")
        self.sums = torch.zeros(4, **f64)
        self.sum_parts = torch.zeros((2, 4), **f64)
        self.scal = torch.zeros(C.sizeof(N.PcgScal) // 8 + 1, **f64)
        self.tol = config.linear_solver.tolerance
        self.max_iter = config.linear_solver.max_iterations
        self.dt = loc.dt
        self.iters = []
        self._args = {}
        labels = [v.config.label for v in loc.lift_volumes]
        self._lift_vectors = tuple(
            loc.currents[labels.index(v.label), :self.n_local] if v.label in labels
            else torch.zeros(self.n_local, **f64)
            for v in config.volumes if not v.disabled)
        # the initial potential of every ghost is its owner's (interface nodes
        # take the smallest material ID's resting value: the owner sees all
        # of its volumes, a ghost may not)
        self.comm.halo(loc.u_ring[0, :loc.n])

    # -- state ----------------------------------------------------------------
    @property
    def step_index(self):
        return self.local.step_index

    @property
    def time(self):
        return self.local.time

    def describe(self):
        p = self.part
        kind = {1: "stencil27", 2: "csr", 3: "sell32", 4: "diasym"}[self.local.op.kind]
        geo = "logical-grid boxes" if p.box is not None else "node coordinates"
        return (f"RCB on {geo} x{self.nranks}; rank-local setup ({kind} local operator); "
                f"NCCL halo ({self.comm.nsend} send / {self.comm.nrecv} recv nodes on rank "
                f"{self.rank}) overlapped with the interior sweep + one 4-sum all-reduce per "
                f"pipelined-PCG iteration, device-resident scalars")

    # -- backend protocol ------------------------------------------------------
    @property
    def x(self):
        return self._x

    @property
    def combo(self):
        return self.local.combo[:self.n_local]

    def lift_currents(self):
        """One current vector per conducting volume of the GLOBAL config (the
        same count and order on every rank, so the halo messages match); a
        volume with no local element contributes zeros (none of this rank's
        owned nodes belongs to it)."""
        return self._lift_vectors

    @property
    def z(self):
        return self.local.ws.z[:self.n_local]

    def m_buffer(self, k):
        n = self.n_local
        return self.local.ws.m[k * n:(k + 1) * n]

    def _sel_args(self, sel):
        b = self._args.get(sel)
        if b is None:
            b = N.CgArgs.from_buffer_copy(self._base)
            b.row_select = sel
            self._args[sel] = b
        return b

    def phase(self, kind, alpha=0.0, beta=0.0, first=0, mbuf=0, sel=3):
        N.check(N.lib().mdx_pcg_phase(N.C.byref(self._sel_args(sel)), kind, 1, alpha, beta,
                                      first, mbuf, N.ptr(self.sums), N.stream_handle()),
                "mdx_pcg_phase")
        self.launches += 2          # phase kernel + partial reduction
        return self.sums.clone()

    def phase_dev(self, kind, mbuf=0, sel=3, part=None):
        out = self.sums if part is None else self.sum_parts[part]
        N.check(N.lib().mdx_pcg_phase_dev(N.C.byref(self._sel_args(sel)), kind, 1,
                                          N.ptr(self.scal), mbuf, N.ptr(out),
                                          N.stream_handle()), "mdx_pcg_phase_dev")
        self.launches += 2

    def combine_parts(self, k):
        import torch

        torch.sum(self.sum_parts[:k], 0, out=self.sums)

    def scalars(self, phase):
        N.check(N.lib().mdx_pcg_scalars(N.ptr(self.sums), N.ptr(self.scal), phase, self.tol,
                                        self.max_iter, N.stream_handle()), "mdx_pcg_scalars")
        self.launches += 1

    def read_scalars(self):
        raw = self.scal.cpu().numpy().tobytes()
        return N.PcgScal.from_buffer_copy(raw[:C.sizeof(N.PcgScal)])

    # -- stepping --------------------------------------------------------------
    def step(self, device_scalars=True):
        loc = self.local
        order, t_next, mask, head, nslot = loc.step_plan()
        l0 = loc.launches
        loc.enqueue_ionic(order, mask, head)
        self.launches += loc.launches - l0
        base = N.CgArgs.from_buffer_copy(loc.solve_args(order, t_next, head, nslot))
        base.row_begin, base.row_end = 0, self.n_local
        base.row_mask = N.ptr(self.row_mask)
        base.row_select = ROW_INTERIOR | ROW_BOUNDARY
        self._base = base
        self._args = {3: base}
        self._x = loc.u_ring[nslot, :self.n_local]
        if device_scalars:
            it, rel, nonfinite = DevicePcgDriver(
                self.comm, self, self.tol, self.max_iter,
                predict=max(self.iters[-1] - 1, 1) if self.iters else 8).solve()
        else:
            it, rel, nonfinite = PipelinedPcgDriver(self.comm, self, self.tol,
                                                    self.max_iter).solve()
        if it < 0:
            raise SolverDivergence(-it, rel)
        if nonfinite:
            raise NonFiniteSolution("linear solve produced non-finite entries")
        if device_scalars:
            self.phase_dev(PH_ACT)
        else:
            self.phase(PH_ACT)
        self.iters.append(it)
        loc.advance_bookkeeping(head, nslot, t_next)
        loc._pending = []
        return it

    # -- outputs ---------------------------------------------------------------
    def potential_local(self):
        return self.local.u_ring[self.local.head, :self.n_local]

    def local_range(self):
        import torch

        u = self.potential_local()[self.owned_idx]
        return torch.stack([u.min(), u.max()])

    def _gather_owned(self, values):
        """Global array of per-owned-node values from every rank."""
        import torch
        import torch.distributed as dist

        k = torch.tensor([self.owned_idx.numel()], device="cuda")
        sizes = [torch.zeros_like(k) for _ in range(self.nranks)]
        dist.all_gather(sizes, k, group=self.comm.group)
        width = int(max(int(s.item()) for s in sizes))
        buf = torch.zeros((2, width), dtype=torch.float64, device="cuda")
        buf[0, :k.item()] = self.owned_global.to(torch.float64)
        buf[1, :k.item()] = values
        parts = [torch.empty_like(buf) for _ in range(self.nranks)]
        dist.all_gather(parts, buf, group=self.comm.group)
        out = np.empty(self.n_global)
        for p, s in zip(parts, sizes):
            h = p.cpu().numpy()
            m = int(s.item())
            out[h[0, :m].astype(np.int64)] = h[1, :m]
        return out

    def gather_potential(self):
        return self._gather_owned(self.potential_local()[self.owned_idx])

    def gather_activation_map(self):
        import torch

        loc = self.local
        fr = loc.frozen[:self.n_local][self.owned_idx].to(torch.float64)
        act = torch.where(fr > 0, loc.act_time[:self.n_local][self.owned_idx],
                          torch.full_like(fr, -1.0))
        return self._gather_owned(act)

    def snapshot_host(self):
        """This rank's state as a pinned host checkpoint payload."""
        import torch

        raw = self.local.checkpoint_payload()
        return torch.frombuffer(bytearray(raw), dtype=torch.uint8).pin_memory()

    def restore_host(self, payload):
        """Restore a snapshot_host payload; returns the bytes moved."""
        n_iters = len(self.iters)
        self.local.restore(payload)
        del self.iters[n_iters:]
        return payload.numel()
