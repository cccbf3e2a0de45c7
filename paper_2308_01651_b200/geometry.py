"""Meshes, structured slabs and fiber fields (host-side data formats).

Mirrors the types the monodomain path consumes from
`/root/reference/pkg/src/monodomain/geometry.py`: `ElementKind` (`:36-48`),
`Mesh` (`:104-173`), `SlabSpec` (`:176-206`), `build_slab_mesh`
(`:219-261`), `nearest_node` (`:264-267`), `FiberField` (`:270-296`) and
`slab_fiber_field` (`:299-331`).  Node and element numbering is identical to
the reference (node id `i + (nx+1)*(j + (ny+1)*k)`, elements x-fastest, VTK
corner order, Kuhn six-tet split), because the device operators are checked
against the reference vector for vector.

Structured slabs additionally carry their lattice shape (`Mesh.lattice`), which
is what lets the device use the class-table stencil operator instead of CSR.
`write_msh` / `import_msh` exchange meshes with the reference in its MSH 2.2
ASCII dialect (`geometry.py:380-517`: 1-based ids, first physical tag =
material id, lower-dimensional elements skipped) - SURVEY.md §8(f) item 3,
so the reference can run the generated config-4 ventricle.  Other MSH
versions and VTK import stay out of scope.
"""

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .errors import (CorruptFile, DegenerateThickness, InvertedElement, NonDivisibleExtent,
                     ZeroSpacing)


class ElementKind(Enum):
    HEX8 = "Hex8"
    TET4 = "Tet4"

    @classmethod
    def from_name(cls, name):
        for kind in cls:
            if kind.value == name:
                return kind
        raise ValueError(f"unknown element kind {name!r}")


NODES_PER_ELEMENT = {ElementKind.HEX8: 8, ElementKind.TET4: 4}

# lattice offsets (dx, dy, dz) of the eight VTK hexahedron corners
HEX_CORNER_OFFSETS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
                      (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))
# Kuhn split of a cube into six tets sharing the c000-c111 diagonal; corners
# are numbered a + 2b + 4c for lattice offset (a, b, c)
KUHN_TETS = ((0, 1, 3, 7), (0, 5, 1, 7), (0, 3, 2, 7),
             (0, 2, 6, 7), (0, 4, 5, 7), (0, 6, 4, 7))

_G = 1.0 / np.sqrt(3.0)
_GAUSS = np.array([(x, y, z) for z in (-_G, _G) for y in (-_G, _G)
                   for x in (-_G, _G)])
_SIGNS = np.array([(2 * a - 1, 2 * b - 1, 2 * c - 1)
                   for (a, b, c) in HEX_CORNER_OFFSETS], dtype=np.float64)


def _hex_ref_gradients():
    out = np.empty((8, 8, 3))
    for p, xi in enumerate(_GAUSS):
        fac = (1.0 + _SIGNS * xi) / 2.0              # (8 corners, 3)
        out[p, :, 0] = _SIGNS[:, 0] / 2.0 * fac[:, 1] * fac[:, 2]
        out[p, :, 1] = _SIGNS[:, 1] / 2.0 * fac[:, 0] * fac[:, 2]
        out[p, :, 2] = _SIGNS[:, 2] / 2.0 * fac[:, 0] * fac[:, 1]
    return out


def tet_volumes6(nodes, tets, chunk=1 << 22):
    """Signed 6 x volume (det of the edge matrix) of every tet, in chunks."""
    out = np.empty(tets.shape[0])
    for b in range(0, tets.shape[0], chunk):
        t = tets[b:b + chunk]
        p0 = nodes[t[:, 0]]
        e1, e2, e3 = nodes[t[:, 1]] - p0, nodes[t[:, 2]] - p0, nodes[t[:, 3]] - p0
        out[b:b + chunk] = (e1[:, 0] * (e2[:, 1] * e3[:, 2] - e2[:, 2] * e3[:, 1])
                            - e1[:, 1] * (e2[:, 0] * e3[:, 2] - e2[:, 2] * e3[:, 0])
                            + e1[:, 2] * (e2[:, 0] * e3[:, 1] - e2[:, 1] * e3[:, 0]))
    return out


def element_jacobians(nodes, elements, kind):
    if kind is ElementKind.TET4:
        return tet_volumes6(nodes, elements)[:, None]
    coords = nodes[elements]
    jac = np.einsum("pak,eaj->epjk", _hex_ref_gradients(), coords)
    return np.linalg.det(jac)


@dataclass
class Mesh:
    """Single-kind conforming mesh with one material ID per element.

    `lattice` is `(nx, ny, nz)` cell counts when the mesh is a structured slab
    numbered exactly like `build_slab_mesh`, else None.
    """

    nodes: np.ndarray
    elements: np.ndarray
    element_kind: ElementKind
    material_ids: np.ndarray
    lattice: tuple = field(default=None, compare=False)
    # logical node grid ((d0, d1, d2), (periodic0, periodic1, periodic2)) with
    # node id = i0 + d0 (i1 + d1 i2), when the generator knows it (ventricle)
    grid: tuple = field(default=None, compare=False)

    def __post_init__(self):
        self.nodes = np.ascontiguousarray(self.nodes, dtype=np.float64)
        self.elements = np.ascontiguousarray(self.elements, dtype=np.int32)
        self.material_ids = np.ascontiguousarray(self.material_ids,
                                                 dtype=np.int32)

    @property
    def num_nodes(self):
        return self.nodes.shape[0]

    @property
    def num_elements(self):
        return self.elements.shape[0]

    def bounding_box(self):
        return self.nodes.min(axis=0), self.nodes.max(axis=0)

    def validate(self):
        n_per = NODES_PER_ELEMENT[self.element_kind]
        if self.elements.ndim != 2 or self.elements.shape[1] != n_per:
            raise ValueError(f"{self.element_kind.value} connectivity must "
                             f"have {n_per} nodes per element")
        if self.material_ids.shape != (self.num_elements,):
            raise ValueError("material_ids must have one entry per element")
        if self.num_elements and (self.elements.min() < 0 or
                                  self.elements.max() >= self.num_nodes):
            raise ValueError("element connectivity references unknown nodes")
        dets = element_jacobians(self.nodes, self.elements, self.element_kind)
        bad = np.flatnonzero((dets <= 0.0).any(axis=1))
        if bad.size:
            raise InvertedElement(
                f"element {bad[0]} has non-positive Jacobian determinant")
        return self

    def with_materials(self, material_ids):
        """Same geometry and lattice, new per-element material IDs."""
        return Mesh(self.nodes, self.elements, self.element_kind,
                    material_ids, lattice=self.lattice, grid=self.grid)


@dataclass(frozen=True)
class SlabSpec:
    extent: tuple
    spacing: float
    element_kind: ElementKind = ElementKind.HEX8

    def __post_init__(self):
        object.__setattr__(self, "extent",
                           tuple(float(e) for e in self.extent))
        if len(self.extent) != 3 or any(e <= 0 for e in self.extent):
            raise ValueError("slab extent must be three positive lengths")
        if self.spacing <= 0:
            raise ZeroSpacing("slab element size must be positive")

    def cells_per_axis(self):
        counts = []
        for length in self.extent:
            n = int(round(length / self.spacing))
            if n < 1 or abs(n * self.spacing - length) > 1e-9 * length:
                raise NonDivisibleExtent(
                    f"extent {length} is not an integer multiple of "
                    f"element size {self.spacing}")
            counts.append(n)
        return tuple(counts)


def lattice_node_id(i, j, k, nx, ny):
    return i + (nx + 1) * (j + (ny + 1) * k)


def build_slab_mesh(spec):
    """Structured slab, material 1 everywhere (reference geometry.py:219)."""
    nx, ny, nz = spec.cells_per_axis()
    h = spec.spacing
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1),
                          np.arange(nx + 1), indexing="ij")
    nodes = np.column_stack([i.ravel() * h, j.ravel() * h, k.ravel() * h])

    # cells x-fastest, then y, then z
    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx),
                             indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    corners = np.column_stack([
        lattice_node_id(ci + a, cj + b, ck + c, nx, ny)
        for (a, b, c) in HEX_CORNER_OFFSETS
    ])
    if spec.element_kind is ElementKind.HEX8:
        elements = corners
    else:
        kuhn = np.column_stack([
            lattice_node_id(ci + (q & 1), cj + ((q >> 1) & 1),
                            ck + ((q >> 2) & 1), nx, ny)
            for q in range(8)
        ])
        elements = np.stack([kuhn[:, list(t)] for t in KUHN_TETS],
                            axis=1).reshape(-1, 4)
    mesh = Mesh(nodes, elements, spec.element_kind,
                np.ones(elements.shape[0], dtype=np.int32),
                lattice=(nx, ny, nz))
    return mesh.validate()


def nearest_node(mesh, point):
    d = mesh.nodes - np.asarray(point, dtype=np.float64)
    return int(np.argmin(np.einsum("ij,ij->i", d, d)))


@dataclass
class FiberField:
    """Orthonormal nodal frame (fiber f0, sheet s0, normal n0)."""

    f0: np.ndarray
    s0: np.ndarray
    n0: np.ndarray

    def __post_init__(self):
        self.f0 = np.ascontiguousarray(self.f0, dtype=np.float64)
        self.s0 = np.ascontiguousarray(self.s0, dtype=np.float64)
        self.n0 = np.ascontiguousarray(self.n0, dtype=np.float64)

    def validate(self):
        for name, arr in (("f0", self.f0), ("s0", self.s0), ("n0", self.n0)):
            if np.abs(np.linalg.norm(arr, axis=1) - 1.0).max(initial=0.0) \
                    > 1e-10:
                raise ValueError(f"{name} is not unit length at every node")
        for a, b, tag in ((self.f0, self.s0, "f0·s0"),
                          (self.f0, self.n0, "f0·n0"),
                          (self.s0, self.n0, "s0·n0")):
            if np.abs(np.einsum("ij,ij->i", a, b)).max(initial=0.0) > 1e-8:
                raise ValueError(f"fiber frame not orthonormal: {tag}")
        return self


def slab_fiber_field(mesh, transmural_axis, endo_angle, epi_angle):
    """Transmurally rotating fibers (reference geometry.py:299-331)."""
    lo, hi = mesh.bounding_box()
    size = hi - lo
    thickness = size[transmural_axis]
    if thickness <= 0.0:
        raise DegenerateThickness(
            f"slab has zero thickness along axis {transmural_axis}")
    in_plane = [a for a in range(3) if a != transmural_axis]
    long_axis = max(in_plane, key=lambda a: (size[a], a))
    e_n = np.eye(3)[transmural_axis]
    e_long = np.eye(3)[long_axis]
    e_perp = np.cross(e_n, e_long)
    phi = (mesh.nodes[:, transmural_axis] - lo[transmural_axis]) / thickness
    ang = np.deg2rad(endo_angle + phi * (epi_angle - endo_angle))
    f0 = np.outer(np.cos(ang), e_long) + np.outer(np.sin(ang), e_perp)
    n0 = np.tile(e_n, (mesh.num_nodes, 1))
    s0 = np.cross(n0, f0)
    return FiberField(f0=f0, s0=s0, n0=n0).validate()


# ---------------------------------------------------------------------------
# MSH 2.2 ASCII exchange with the reference (geometry.py:380-517 there)
# ---------------------------------------------------------------------------

_MSH_TYPE = {ElementKind.TET4: 4, ElementKind.HEX8: 5}
_MSH_KIND = {4: ElementKind.TET4, 5: ElementKind.HEX8}
_MSH_LOWER_DIM = {1, 2, 3, 15}          # lines, triangles, quads, points: skipped


def write_msh(mesh, path):
    """MSH 2.2 ASCII: 1-based node/element ids, one physical tag (material id),
    coordinates with 17 significant digits (round-trips fp64 exactly)."""
    etype = _MSH_TYPE[mesh.element_kind]
    n, e = mesh.num_nodes, mesh.num_elements
    with open(path, "w", encoding="ascii") as fh:
        fh.write("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n")
        fh.write(f"$Nodes\n{n}\n")
        ids = np.arange(1, n + 1)
        np.savetxt(fh, np.column_stack([ids, mesh.nodes]), fmt=["%d", "%.17g", "%.17g", "%.17g"])
        fh.write(f"$EndNodes\n$Elements\n{e}\n")
        cols = np.column_stack([np.arange(1, e + 1), np.full(e, etype), np.ones(e, dtype=np.int64),
                                mesh.material_ids.astype(np.int64),
                                mesh.elements.astype(np.int64) + 1])
        np.savetxt(fh, cols, fmt="%d")
        fh.write("$EndElements\n")


def import_msh(path, scaling_factor=1.0):
    """Read an MSH 2.x ASCII volume mesh (tets or hexes, not mixed); the first
    physical tag of each volume element becomes its material id.  Raises
    CorruptFile on anything malformed."""
    with open(path, encoding="ascii") as fh:
        lines = fh.read().split("\n")

    def section(name):
        try:
            a = lines.index(f"${name}")
            b = lines.index(f"$End{name}", a)
        except ValueError:
            raise CorruptFile(f"MSH file lacks a ${name} section")
        return lines[a + 1:b]

    if "$MeshFormat" in lines and not section("MeshFormat")[0].split()[0].startswith("2."):
        raise CorruptFile("only MSH format 2.x is supported")
    body = section("Nodes")
    try:
        count = int(body[0])
        tab = np.array([ln.split() for ln in body[1:count + 1]], dtype=np.float64)
    except (ValueError, IndexError):
        raise CorruptFile("malformed $Nodes section")
    if tab.shape != (count, 4):
        raise CorruptFile("node lines must be 'id x y z'")
    node_ids = tab[:, 0].astype(np.int64)
    order = np.argsort(node_ids)
    if np.unique(node_ids).size != count:
        raise CorruptFile("duplicate node ids")
    body = section("Elements")
    conn, tags, kind = [], [], None
    try:
        ecount = int(body[0])
        rows = [ln.split() for ln in body[1:ecount + 1]]
    except ValueError:
        raise CorruptFile("malformed $Elements section")
    for parts in rows:
        etype, ntags = int(parts[1]), int(parts[2])
        if etype in _MSH_LOWER_DIM:
            continue
        if etype not in _MSH_KIND:
            raise CorruptFile(f"unsupported MSH element type {etype}")
        k = _MSH_KIND[etype]
        if kind is None:
            kind = k
        elif k is not kind:
            raise CorruptFile("mesh mixes element types")
        if ntags < 1:
            raise CorruptFile("volume element without a physical tag")
        tags.append(int(parts[3]))
        conn.append([int(x) for x in parts[3 + ntags:]])
    if kind is None:
        raise CorruptFile("no volume elements")
    conn = np.asarray(conn, dtype=np.int64)
    if conn.shape[1] != NODES_PER_ELEMENT[kind]:
        raise CorruptFile("wrong node count per element")
    pos = np.searchsorted(node_ids[order], conn)
    if (pos >= count).any() or (node_ids[order][np.minimum(pos, count - 1)] != conn).any():
        raise CorruptFile("element references an unknown node id")
    mesh = Mesh(tab[:, 1:] * float(scaling_factor), order[pos].astype(np.int32), kind,
                np.asarray(tags, dtype=np.int32))
    mesh.validate()
    return mesh


read_msh = import_msh
