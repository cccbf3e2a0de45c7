"""Output formats at the record stride: CSV time series and legacy VTK.

Byte-compatible restatement of `/root/reference/pkg/src/monodomain/outputs.py`
(`OutputConfig` `:19-33`, `write_csv` `:39-50`, `write_zero_d_trace`
`:53-63`, `write_vtk` `:66-119`): `%.8e` numbers, `t,u_min,u_max,probe_i`
header, VTK cell types 12 (hex) / 10 (tet), material IDs as cell data.
These are host-side file writers, fed from device read-backs at the output
stride; they are not on the per-step path.
"""

from dataclasses import dataclass

import numpy as np

from .errors import MonodomainError


class IoFailure(MonodomainError):
    """An output file could not be written."""


class LengthMismatch(MonodomainError):
    """A nodal field does not match the mesh node count."""


@dataclass
class OutputConfig:
    enable_field_output: bool = False
    field_stem: str = "solution"
    enable_csv: bool = False
    csv_path: str = "trace.csv"
    stride: int = 1
    probe_points: tuple = ()

    def __post_init__(self):
        if self.stride < 1:
            raise ValueError("output stride must be >= 1")


def _fmt(v):
    return f"{v:.8e}"


def _write(path, lines, what):
    try:
        with open(path, "w", encoding="ascii", newline="\n") as fh:
            fh.writelines(lines)
    except OSError as exc:
        raise IoFailure(f"cannot write {what} {path}: {exc}") from exc


def write_csv(path, rows, probe_count=0):
    header = "t,u_min,u_max" + "".join(f",probe_{i}" for i in range(probe_count))
    lines = [header + "\n"] + [",".join(_fmt(v) for v in r) + "\n" for r in rows]
    _write(path, lines, "CSV")


def write_zero_d_trace(path, trace):
    nv = trace.shape[1] - 2
    header = "t,u" + "".join(f",w{i + 1}" for i in range(nv))
    lines = [header + "\n"] + [",".join(_fmt(v) for v in r) + "\n" for r in trace]
    _write(path, lines, "CSV")


_CELL_TYPE = {"Hex8": 12, "Tet4": 10}


def write_vtk(path, mesh, point_fields=None):
    point_fields = point_fields or {}
    n = mesh.nodes.shape[0]
    ne = mesh.elements.shape[0]
    for name, values in point_fields.items():
        if np.asarray(values).shape[0] != n:
            raise LengthMismatch(f"field {name!r} has {np.asarray(values).shape[0]} "
                                 f"values for {n} nodes")
    npe = mesh.elements.shape[1]
    out = ["# vtk DataFile Version 3.0\n", "monodomain output\n", "ASCII\n",
           "DATASET UNSTRUCTURED_GRID\n", f"POINTS {n} double\n"]
    out += [f"{_fmt(x)} {_fmt(y)} {_fmt(z)}\n" for x, y, z in mesh.nodes]
    out.append(f"CELLS {ne} {ne * (1 + npe)}\n")
    out += [f"{npe} " + " ".join(str(c) for c in conn) + "\n" for conn in mesh.elements]
    out.append(f"CELL_TYPES {ne}\n")
    ct = _CELL_TYPE[mesh.element_kind.value]
    out += [f"{ct}\n"] * ne
    out.append(f"CELL_DATA {ne}\n")
    out.append("SCALARS material_id int 1\nLOOKUP_TABLE default\n")
    out += [f"{m}\n" for m in mesh.material_ids]
    if point_fields:
        out.append(f"POINT_DATA {n}\n")
        for name, values in point_fields.items():
            values = np.asarray(values)
            if values.ndim == 2 and values.shape[1] == 3:
                out.append(f"VECTORS {name} double\n")
                out += [f"{_fmt(v[0])} {_fmt(v[1])} {_fmt(v[2])}\n" for v in values]
            else:
                out.append(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
                out += [f"{_fmt(v)}\n" for v in values]
    _write(path, out, "VTK")
