"""P1/Q1 finite-element operators, assembled on the device.

Mirror of `/root/reference/pkg/src/monodomain/fem.py`: quadrature tables
(`:36-85`), `ConductivitySet` (`:93-128`), `diffusion_tensor` (`:131-144`),
`FeSpace` (`:152-239`), pattern (`:242-259`), assembly front ends
(`:434-486`) and `ici_lift` (`:489-504`).

The element integrals and the scatter run in `csrc/assembly.cu` (compiled
with `--fmad=false`), so every assembled entry is bit-identical to the
reference.  Two device forms come out of the same element matrices:

* CSR values on the reference's pattern (any mesh);
* 27-point stencil rows for structured hex slabs, which `StencilOperator`
  compresses into per-node class ids + class tables (matrix-free apply).

The public `assemble_mass` / `assemble_stiffness` return scipy CSR matrices
(drop-in for callers of the reference API); the tissue solver keeps
everything on the device.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .errors import KeyMismatch, MissingConductivity, NonOrthonormalFrame
from .geometry import ElementKind, HEX_CORNER_OFFSETS, lattice_node_id

# ---------------------------------------------------------------------------
# Reference elements (fem.py:36-85): same expressions, hence the same bits
# ---------------------------------------------------------------------------


def _hex_tables():
    g = 1.0 / np.sqrt(3.0)
    pts = [(x, y, z) for z in (-g, g) for y in (-g, g) for x in (-g, g)]
    signs = [(2 * a - 1, 2 * b - 1, 2 * c - 1) for (a, b, c) in HEX_CORNER_OFFSETS]
    weights = np.ones(8)
    values = np.empty((8, 8))
    grads = np.empty((8, 8, 3))
    for p, xi in enumerate(pts):
        for a, s in enumerate(signs):
            f = [(1.0 + float(s[d]) * xi[d]) / 2.0 for d in range(3)]
            values[p, a] = f[0] * f[1] * f[2]
            grads[p, a, 0] = float(s[0]) / 2.0 * f[1] * f[2]
            grads[p, a, 1] = float(s[1]) / 2.0 * f[0] * f[2]
            grads[p, a, 2] = float(s[2]) / 2.0 * f[0] * f[1]
    return weights, values, grads


def _tet_tables():
    a, b = 0.5854101966249685, 0.1381966011250105
    values = np.array([(a, b, b, b), (b, a, b, b), (b, b, a, b), (b, b, b, a)])
    weights = np.full(4, 1.0 / 24.0)
    g = np.array([(-1.0, -1.0, -1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                  (0.0, 0.0, 1.0)])
    return weights, values, np.broadcast_to(g, (4, 4, 3)).copy()


QUADRATURE = {ElementKind.HEX8: _hex_tables(), ElementKind.TET4: _tet_tables()}


def _kind_of(mesh):
    kind = mesh.element_kind
    return kind if isinstance(kind, ElementKind) else ElementKind.from_name(kind.value)


# ---------------------------------------------------------------------------
# Conductivities
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SubdomainConductivity:
    sigma_l: float = 0.0
    sigma_t: float = 0.0
    sigma_n: float = 0.0
    disabled: bool = False

    def __post_init__(self):
        if not self.disabled and min(self.sigma_l, self.sigma_t, self.sigma_n) < 0.0:
            raise ValueError("conductivities must be non-negative")


@dataclass
class ConductivitySet:
    entries: dict = field(default_factory=dict)

    def add(self, material_id, sigma_l, sigma_t, sigma_n, disabled=False):
        self.entries[int(material_id)] = SubdomainConductivity(
            sigma_l, sigma_t, sigma_n, disabled)
        return self

    def __contains__(self, material_id):
        return int(material_id) in self.entries

    def __getitem__(self, material_id):
        return self.entries[int(material_id)]

    def disabled_ids(self):
        return {m for m, c in self.entries.items() if c.disabled}


def diffusion_tensor(sigma, f0, s0, n0):
    frame = np.array([f0, s0, n0], dtype=np.float64)
    if np.abs(frame @ frame.T - np.eye(3)).max() > 1e-6:
        raise NonOrthonormalFrame("fiber frame is not orthonormal within 1e-6")
    sl, st, sn = sigma
    return (sl * np.outer(frame[0], frame[0]) + st * np.outer(frame[1], frame[1])
            + sn * np.outer(frame[2], frame[2]))


# ---------------------------------------------------------------------------
# FE space (host bookkeeping: pattern, DOF/material adjacency)
# ---------------------------------------------------------------------------


class FeSpace:
    def __init__(self, mesh, degree=1):
        if degree != 1:
            raise ValueError(f"only degree-1 elements are supported, got degree {degree}")
        self.mesh = mesh
        self.degree = degree
        self.dof_coords = mesh.nodes
        self._pattern = None
        self._incidence = None
        self._adjacency = None

    @property
    def num_dofs(self):
        return self.mesh.nodes.shape[0]

    def pattern(self):
        """(indptr int64, indices int32) of all node pairs sharing an element.

        Sorted unique (row, column) keys: on the device when one is visible
        (the 960 M candidate pairs of the 10 M-node ventricle sort in about a
        second there, minutes with numpy), else on the host."""
        if self._pattern is None:
            n = self.num_dofs
            torch = _torch_if_cuda()
            if torch is not None:
                e = torch.from_numpy(np.ascontiguousarray(self.mesh.elements)).cuda().long()
                nl = e.shape[1]
                keys = (e.repeat_interleave(nl, dim=1) * n + e.repeat(1, nl)).reshape(-1)
                del e
                keys = torch.unique(keys)                      # sorted
                rows = torch.div(keys, n, rounding_mode="floor")
                indptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
                indptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
                cols = (keys - rows * n).to(torch.int32)
                self._pattern = (indptr.cpu().numpy(), cols.cpu().numpy())
            else:
                e = np.asarray(self.mesh.elements, dtype=np.int64)
                nl = e.shape[1]
                keys = (np.repeat(e, nl, axis=1) * n + np.tile(e, (1, nl))).ravel()
                keys = np.unique(keys)
                rows = keys // n
                indptr = np.zeros(n + 1, dtype=np.int64)
                np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
                self._pattern = (indptr, (keys % n).astype(np.int32))
        return self._pattern

    def incidence(self):
        """Per node: incident (element, local corner), ascending element."""
        if self._incidence is None:
            e = np.asarray(self.mesh.elements)
            nl = e.shape[1]
            torch = _torch_if_cuda()
            if torch is not None:
                flat = torch.from_numpy(np.ascontiguousarray(e).ravel()).cuda()
                _, order = torch.sort(flat, stable=True)
                ptr = torch.zeros(self.num_dofs + 1, dtype=torch.int64, device="cuda")
                ptr[1:] = torch.cumsum(torch.bincount(flat, minlength=self.num_dofs), 0)
                self._incidence = (ptr.cpu().numpy(), (order // nl).to(torch.int32).cpu().numpy(),
                                   (order % nl).to(torch.int8).cpu().numpy())
            else:
                flat = e.ravel()
                order = np.argsort(flat, kind="stable")
                ptr = np.zeros(self.num_dofs + 1, dtype=np.int64)
                np.cumsum(np.bincount(flat, minlength=self.num_dofs), out=ptr[1:])
                self._incidence = (ptr, (order // nl).astype(np.int32),
                                   (order % nl).astype(np.int8))
        return self._incidence

    def _dof_materials(self):
        if self._adjacency is None:
            e = self.mesh.elements
            pairs = np.unique(np.column_stack(
                [e.ravel(), np.repeat(self.mesh.material_ids, e.shape[1])]), axis=0)
            indptr = np.zeros(self.num_dofs + 1, dtype=np.int64)
            np.add.at(indptr, pairs[:, 0] + 1, 1)
            np.cumsum(indptr, out=indptr)
            self._adjacency = (indptr, pairs[:, 1].astype(np.int32))
        return self._adjacency

    def material_ids(self):
        return np.unique(self.mesh.material_ids)

    def dofs_in_subdomain(self, material_id):
        """Sorted unique nodes of the elements of one material (a node mask:
        the same set as np.unique, in linear time)."""
        mask = self.mesh.material_ids == material_id
        hit = np.zeros(self.num_dofs, dtype=bool)
        hit[self.mesh.elements[mask].ravel()] = True
        return np.flatnonzero(hit)

    def inactive_dof_mask(self, disabled_material_ids):
        """DOFs adjacent only to disabled materials (fem.py:225-239)."""
        disabled = {int(m) for m in disabled_material_ids}
        if not disabled:
            return np.zeros(self.num_dofs, dtype=bool)
        indptr, mats = self._dof_materials()
        active = np.array([m for m in self.material_ids() if int(m) not in disabled],
                          dtype=np.int32)
        owner = np.repeat(np.arange(self.num_dofs), np.diff(indptr))
        touches = np.zeros(self.num_dofs, dtype=bool)
        touches[owner[np.isin(mats, active)]] = True
        return (np.diff(indptr) > 0) & ~touches


# ---------------------------------------------------------------------------
# Device assembly
# ---------------------------------------------------------------------------


def _torch():
    import torch

    return torch


def _torch_if_cuda():
    """torch when a CUDA device is visible (setup-time sorting), else None."""
    try:
        import torch
    except ImportError:
        return None
    return torch if torch.cuda.is_available() else None


class DeviceMesh:
    """Mesh + fibers uploaded once; element matrices computed on demand."""

    def __init__(self, mesh, fibers=None):
        torch = _torch()
        self.mesh = mesh
        self.kind = _kind_of(mesh)
        self.nl = mesh.elements.shape[1]
        self.n = mesh.nodes.shape[0]
        self.ne = mesh.elements.shape[0]
        self.nodes = torch.from_numpy(np.ascontiguousarray(mesh.nodes, np.float64)).cuda()
        self.elements = torch.from_numpy(
            np.ascontiguousarray(mesh.elements, np.int32)).cuda()
        if fibers is not None:
            self.f0 = torch.from_numpy(np.ascontiguousarray(fibers.f0, np.float64)).cuda()
            self.s0 = torch.from_numpy(np.ascontiguousarray(fibers.s0, np.float64)).cuda()
        else:
            self.f0 = self.s0 = None

    def element_matrices(self, sigma_rows=None, sigmas=None, want_k=True, want_m=True):
        """(K_local, M_local) device tensors of shape (E, nl, nl)."""
        torch = _torch()
        w, basis, grad = QUADRATURE[self.kind]
        keep = []
        wh, wp = N.host_doubles(w)
        bh, bp = N.host_doubles(basis)
        gh, gp = N.host_doubles(grad)
        keep += [wh, bh, gh]
        K = torch.empty((self.ne, self.nl, self.nl), dtype=torch.float64,
                        device="cuda") if want_k else None
        M = torch.empty((self.ne, self.nl, self.nl), dtype=torch.float64,
                        device="cuda") if want_m else None
        a = N.AssemblyArgs()
        a.n_elem = self.ne
        a.nl = self.nl
        a.nq = w.size
        a.nodes = N.ptr(self.nodes)
        a.elements = N.ptr(self.elements)
        a.quad_w, a.quad_basis, a.quad_grad = wp, bp, gp
        sr = sg = None
        if want_k:
            sr = torch.from_numpy(np.ascontiguousarray(sigma_rows, np.int32)).cuda()
            sg = torch.from_numpy(np.ascontiguousarray(
                np.asarray(sigmas, np.float64).reshape(-1, 3))).cuda()
            a.sigma_row = N.ptr(sr)
            a.sigmas = N.ptr(sg) if sg.numel() else None
            a.f0 = N.ptr(self.f0)
            a.s0 = N.ptr(self.s0)
        a.K_local = N.ptr(K)
        a.M_local = N.ptr(M)
        N.check(N.lib().mdx_assemble_local(N.C.byref(a), N.stream_handle()),
                "mdx_assemble_local")
        return K, M

    def include_mask(self, materials):
        torch = _torch()
        if materials is None:
            return None
        wanted = np.array(sorted(int(m) for m in materials), dtype=np.int32)
        inc = np.isin(self.mesh.material_ids, wanted).astype(np.uint8)
        return torch.from_numpy(inc).cuda()

    def csr_values(self, space, local, include=None):
        torch = _torch()
        indptr, indices = space.pattern()
        ptr_, elem, loc = space.incidence()
        dev = getattr(self, "_csr_dev", None)
        if dev is None:
            dev = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda()
                        for x in (indptr, indices, ptr_, elem, loc))
            self._csr_dev = dev
        d_indptr, d_indices, d_ptr, d_elem, d_loc = dev
        data = torch.empty(indices.size, dtype=torch.float64, device="cuda")
        N.check(N.lib().mdx_scatter_csr(
            self.n, self.nl, N.ptr(self.elements), N.ptr(d_ptr), N.ptr(d_elem),
            N.ptr(d_loc), N.ptr(include), N.ptr(local), N.ptr(d_indptr),
            N.ptr(d_indices), N.ptr(data), N.stream_handle()), "mdx_scatter_csr")
        return data

    def stencil_rows(self, lattice, local, include=None):
        torch = _torch()
        nx, ny, nz = lattice
        rows = torch.empty((self.n, 27), dtype=torch.float64, device="cuda")
        N.check(N.lib().mdx_stencil_rows(nx, ny, nz, N.ptr(include), N.ptr(local),
                                         N.ptr(rows), N.stream_handle()),
                "mdx_stencil_rows")
        return rows


def _sigma_table(space, conductivities):
    """Per-element conductivity row (-1 = no conduction), as fem.py:459-475."""
    mesh = space.mesh
    table, row_of = [], {}
    for mat in space.material_ids():
        mat = int(mat)
        if mat not in conductivities:
            raise MissingConductivity(mat)
        entry = conductivities[mat]
        if entry.disabled:
            row_of[mat] = -1
        else:
            row_of[mat] = len(table)
            table.append((entry.sigma_l, entry.sigma_t, entry.sigma_n))
    mats = np.asarray(mesh.material_ids)
    keys = np.array(sorted(row_of), dtype=np.int64)
    vals = np.array([row_of[k] for k in keys], dtype=np.int32)
    rows = vals[np.searchsorted(keys, mats)]
    return rows, np.asarray(table, dtype=np.float64).reshape(-1, 3)


def _to_scipy(space, data):
    indptr, indices = space.pattern()
    n = space.num_dofs
    return sp.csr_matrix((data.cpu().numpy(), indices.copy(), indptr.copy()),
                         shape=(n, n))


def assemble_mass(space, subdomain_filter=None):
    """Consistent mass matrix (optionally restricted), as scipy CSR."""
    dm = DeviceMesh(space.mesh)
    _, M = dm.element_matrices(want_k=False)
    inc = dm.include_mask(subdomain_filter)
    return _to_scipy(space, dm.csr_values(space, M, inc))


def assemble_stiffness(space, conductivities, fibers):
    """Anisotropic stiffness matrix, as scipy CSR."""
    rows, table = _sigma_table(space, conductivities)
    dm = DeviceMesh(space.mesh, fibers)
    K, _ = dm.element_matrices(rows, table, want_m=False)
    return _to_scipy(space, dm.csr_values(space, K))


def ici_lift(per_subdomain_mass, nodal_currents):
    """sum_i M^i @ I^i over subdomains (fem.py:489-504)."""
    if set(per_subdomain_mass) != set(nodal_currents):
        raise KeyMismatch(
            f"mass matrices cover materials {sorted(per_subdomain_mass)} "
            f"but currents cover {sorted(nodal_currents)}")
    result = None
    for key, matrix in per_subdomain_mass.items():
        term = matrix @ nodal_currents[key]
        result = term if result is None else result + term
    return result


def detect_lattice(mesh):
    """(nx, ny, nz) if `mesh` is numbered exactly like a structured hex slab."""
    if _kind_of(mesh) is not ElementKind.HEX8:
        return None
    lat = getattr(mesh, "lattice", None)
    if lat is not None:
        return tuple(lat)
    nodes = mesh.nodes
    axes = [np.unique(nodes[:, d]) for d in range(3)]
    nx, ny, nz = (len(a) - 1 for a in axes)
    if min(nx, ny, nz) < 1 or (nx + 1) * (ny + 1) * (nz + 1) != nodes.shape[0] \
            or mesh.elements.shape[0] != nx * ny * nz:
        return None
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1),
                          indexing="ij")
    expect = np.column_stack([axes[0][i.ravel()], axes[1][j.ravel()], axes[2][k.ravel()]])
    if not np.array_equal(expect, nodes):
        return None
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    conn = np.column_stack([lattice_node_id(ci + a, cj + b, ck + c, nx, ny)
                            for (a, b, c) in HEX_CORNER_OFFSETS])
    if not np.array_equal(conn, mesh.elements):
        return None
    return (nx, ny, nz)
