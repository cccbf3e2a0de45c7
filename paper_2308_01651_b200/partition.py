"""Mesh partition for the multi-GPU step: recursive coordinate bisection and
rank-local sub-problems.

Host logic only (numpy), shared by the GPU solver (distributed.py) and the
CPU multi-rank tests.

Partition.  `rcb(points, nparts)` bisects the node set recursively at the
weighted median of its longest axis (part counts split as k//2 : k - k//2,
so any rank count works).  On meshes that carry their logical grid
(`Mesh.grid`: structured slabs, the config-4 ventricle) the coordinates
bisected are the logical indices, so every part is a box of the logical
grid; otherwise the physical node coordinates.

Local problem.  A rank owns its part's nodes.  Its local mesh holds every
element touching an owned node (in ascending global element order, so the
assembled rows of the owned nodes are the reference's rows bit for bit) and
their nodes: owned + ghosts.  On a logical grid the local node set is the
part's box grown by one layer (clipped to the grid, wrapped across a periodic
axis) together with every element inside it, numbered lexicographically in
the box: the couplings keep constant index offsets, so the local operator
compresses to diagonals exactly like the global one.  Elsewhere local nodes
are numbered in ascending global order.

Halo.  For every peer: the local indices this rank sends (owned nodes that
are ghosts there) and receives (ghosts it owns), both in ascending global
order, so the two sides agree without a handshake.
"""

from dataclasses import dataclass, field

import numpy as np


def rcb(points, nparts, planes=False):
    """Part id (0..nparts-1) of every point: recursive coordinate bisection.

    Deterministic: ties along the cut axis are broken by point index.  With
    `planes` (integer logical coordinates) a cut never splits a plane: it
    falls between the two coordinate values closest to the proportional
    split, so every part is a box of the grid."""
    points = np.asarray(points, dtype=np.float64)
    n = points.shape[0]
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    if nparts > n:
        raise ValueError(f"{nparts} parts exceed the {n} points")
    part = np.empty(n, dtype=np.int32)

    def split(idx, k, base):
        if k == 1:
            part[idx] = base
            return
        sub = points[idx]
        axis = int(np.argmax(sub.max(axis=0) - sub.min(axis=0)))
        k1 = k // 2
        if planes:
            vals, counts = np.unique(sub[:, axis], return_counts=True)
            below = np.cumsum(counts)[:-1]                    # points below each cut
            if below.size == 0:
                raise ValueError(f"cannot cut {idx.size} points into {k} boxes")
            j = int(np.argmin(np.abs(below - idx.size * k1 / k)))
            left = sub[:, axis] < vals[j + 1]
            split(idx[left], k1, base)
            split(idx[~left], k - k1, base + k1)
            return
        order = np.lexsort((idx, sub[:, axis]))
        cut = int(round(idx.size * k1 / k))
        split(idx[order[:cut]], k1, base)
        split(idx[order[cut:]], k - k1, base + k1)

    split(np.arange(n), nparts, 0)
    return part


def grid_of(mesh):
    """(dims, periodic) of the mesh's logical node grid (node id = i0 + d0 (i1
    + d1 i2)), or None."""
    g = getattr(mesh, "grid", None)
    if g is not None:
        return tuple(g[0]), tuple(bool(p) for p in g[1])
    lat = getattr(mesh, "lattice", None)
    if lat is None:
        from .fem import detect_lattice

        lat = detect_lattice(mesh)
    if lat is not None:
        return tuple(d + 1 for d in lat), (False, False, False)
    return None


def grid_coords(dims, ids):
    d0, d1, _ = dims
    ids = np.asarray(ids, dtype=np.int64)
    return np.stack([ids % d0, (ids // d0) % d1, ids // (d0 * d1)], axis=1)


def partition(mesh, nparts):
    """Owner rank of every node: RCB on the logical grid when the mesh has
    one, else on the node coordinates."""
    g = grid_of(mesh)
    if g is not None:
        pts = grid_coords(g[0], np.arange(mesh.nodes.shape[0])).astype(np.float64)
        return rcb(pts, nparts, planes=True)
    return rcb(mesh.nodes, nparts)


@dataclass
class LocalPart:
    rank: int
    nranks: int
    nodes: np.ndarray           # global id of each local node (local order)
    owned: np.ndarray           # bool per local node
    elements: np.ndarray        # global ids of the local elements, ascending
    conn: np.ndarray            # local connectivity (n_elem, nl) int32
    send: dict = field(default_factory=dict)   # peer -> local indices (sorted by global id)
    recv: dict = field(default_factory=dict)   # peer -> local indices (sorted by global id)
    box: tuple = None           # logical box (lo, hi, dims, periodic) when on a grid

    @property
    def n_local(self):
        return self.nodes.size

    @property
    def n_owned(self):
        return int(self.owned.sum())

    def owned_local(self):
        """Local indices of the owned nodes, in ascending global order."""
        idx = np.flatnonzero(self.owned)
        return idx[np.argsort(self.nodes[idx], kind="stable")]


def _box_nodes(lo, hi, dims, periodic):
    """Global ids of the nodes of a logical box [lo, hi) (hi - lo per axis may
    wrap a periodic axis), lexicographic in the box (axis 0 fastest)."""
    axes = []
    for a in range(3):
        r = np.arange(lo[a], hi[a])
        axes.append(r % dims[a] if periodic[a] else r)
    i2, i1, i0 = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return (i0 + dims[0] * (i1 + dims[1] * i2)).ravel().astype(np.int64)


def _grown_box(coords, dims, periodic):
    """[lo, hi) of the owned coordinates grown by one node per side (clipped,
    or wrapped on a periodic axis when the part does not span it)."""
    lo = np.empty(3, np.int64)
    hi = np.empty(3, np.int64)
    for a in range(3):
        c = np.unique(coords[:, a])
        if periodic[a] and c.size < dims[a]:
            # the owned range may itself wrap: start after the largest gap
            gaps = np.diff(np.concatenate([c, [c[0] + dims[a]]]))
            k = int(np.argmax(gaps))
            start = int(c[(k + 1) % c.size])
            length = dims[a] - int(gaps[k]) + 1
            lo[a], hi[a] = start - 1, start + length + 1
            if hi[a] - lo[a] > dims[a]:
                lo[a], hi[a] = 0, dims[a]
        else:
            lo[a] = max(int(c.min()) - 1, 0)
            hi[a] = min(int(c.max()) + 2, dims[a])
    return lo, hi


def build_part(mesh, owner, rank):
    """The rank-local sub-problem of `owner` (one part id per node)."""
    owner = np.asarray(owner)
    nranks = int(owner.max()) + 1
    el = np.asarray(mesh.elements)
    n = mesh.nodes.shape[0]
    own = owner == rank
    touch = own[el].any(axis=1)
    g = grid_of(mesh)
    box = None
    if g is not None:
        dims, periodic = g
        lo, hi = _grown_box(grid_coords(dims, np.flatnonzero(own)), dims, periodic)
        nodes = _box_nodes(lo, hi, dims, periodic)
        local_of = np.full(n, -1, np.int64)
        local_of[nodes] = np.arange(nodes.size)
        inside = (local_of[el] >= 0).all(axis=1)
        if not (inside | ~touch).all():
            raise AssertionError("an element of an owned node leaves the grown box")
        elements = np.flatnonzero(inside)
        box = (tuple(lo), tuple(hi), dims, periodic)
    else:
        elements = np.flatnonzero(touch)
        nodes = np.unique(el[elements].ravel()).astype(np.int64)
        local_of = np.full(n, -1, np.int64)
        local_of[nodes] = np.arange(nodes.size)
    conn = local_of[el[elements]].astype(np.int32)
    owned = own[nodes]
    # ghosts: local nodes owned elsewhere that an owned node couples to
    coupled = np.zeros(nodes.size, bool)
    owned_el = owned[conn].any(axis=1)
    coupled[conn[owned_el].ravel()] = True
    ghosts = coupled & ~owned
    recv = {}
    for q in np.unique(owner[nodes[ghosts]]):
        li = np.flatnonzero(ghosts & (owner[nodes] == q))
        recv[int(q)] = li[np.argsort(nodes[li], kind="stable")]
    return LocalPart(rank, nranks, nodes, owned, elements, conn, {}, recv, box)


def halo_plans(mesh, owner):
    """LocalPart of every rank with matching send lists (host-side, used by
    every rank to derive its own send lists without communication)."""
    parts = [build_part(mesh, owner, r) for r in range(int(np.max(owner)) + 1)]
    for p in parts:
        local_of = {int(g): i for i, g in enumerate(p.nodes)}
        for q in parts:
            if q.rank == p.rank or p.rank not in q.recv:
                continue
            want = q.nodes[q.recv[p.rank]]
            p.send[q.rank] = np.array([local_of[int(g)] for g in want], np.int64)
    return parts


def send_lists(mesh, owner, part):
    """This rank's send lists: for every peer q, the owned nodes that are
    ghosts of q (ascending global id).  Computed from q's ghost set, which
    every rank can derive from the mesh and the owner array."""
    owner = np.asarray(owner)
    el = np.asarray(mesh.elements)
    rank = part.rank
    own_me = owner == rank
    # elements that touch one of my nodes and a node of q: my nodes on them
    # are coupled to q's owned nodes, i.e. ghosts of q
    local_of = np.full(mesh.nodes.shape[0], -1, np.int64)
    local_of[part.nodes] = np.arange(part.nodes.size)
    mine_el = el[own_me[el].any(axis=1)]
    out = {}
    for q in range(part.nranks):
        if q == rank:
            continue
        e_q = mine_el[(owner[mine_el] == q).any(axis=1)]
        if e_q.size == 0:
            continue
        g = np.unique(e_q.ravel())
        g = g[own_me[g]]
        out[q] = local_of[g]
    return out
