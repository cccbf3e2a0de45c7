"""C-ABI boundary checks that need no GPU.

libmdx.so must load, export every entry point include/mdx.h declares, and
the ctypes struct layouts must match the header's C layout (checked by
compiling a tiny offsetof() probe with gcc against include/mdx.h).
Product entry points must refuse to run without a device (no CPU fallback).
"""

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mdx.h"


@pytest.fixture(scope="module")
def built():
    from paper_2308_01651_b200 import native_build

    native_build.build()
    return native_build.LIB


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(mdx_\w+)\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = header_functions()
    for must in ("mdx_ionic_advance", "mdx_ionic_advance_rl", "mdx_ionic_current", "mdx_ionic_point_rates",
                 "mdx_tissue_ionic", "mdx_tissue_prep", "mdx_pcg_solve", "mdx_spmv",
                 "mdx_assemble_local", "mdx_scatter_csr", "mdx_stencil_rows",
                 "mdx_pace_cells"):
        assert must in names


def test_library_exports_every_header_symbol(built):
    lib = C.CDLL(str(built))
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(built)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (mdx_\w+)", out))
    assert set(header_functions()) <= exported


def test_ctypes_binding_covers_header(built):
    from paper_2308_01651_b200 import _native

    assert set(header_functions()) == set(_native.EXPORTED_SYMBOLS)
    lib = _native.load_library(built)
    assert lib.mdx_abi_version() == _native.ABI_VERSION == 5
    assert lib.mdx_ionic_num_vars(_native.MODEL_TTP06) == 18
    assert lib.mdx_ionic_num_vars(_native.MODEL_BUENO_OROVIO) == 3
    assert lib.mdx_ionic_num_vars(_native.MODEL_ALIEV_PANFILOV) == 1
    assert lib.mdx_ionic_num_params(_native.MODEL_TTP06) == 50
    assert lib.mdx_ionic_num_vars(99) == -1


def test_sm100a_cubin_embedded(built):
    out = subprocess.run(["cuobjdump", "--list-elf", str(built)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


STRUCTS = {
    "mdx_tissue_ionic_args": "TissueIonicArgs",
    "mdx_operator": "Operator",
    "mdx_cg_args": "CgArgs",
    "mdx_assembly_args": "AssemblyArgs",
    "mdx_pace_args": "PaceArgs",
    "mdx_pcg_scal": "PcgScal",
}


def test_struct_layouts_match_header(tmp_path):
    from paper_2308_01651_b200 import _native

    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"',
             "int main(void) {"]
    for cname, pyname in STRUCTS.items():
        cls = getattr(_native, pyname)
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, pyname in STRUCTS.items():
        cls = getattr(_native, pyname)
        assert int(got[f"{cname} size"]) == C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, \
                f"{cname}.{fname}"


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2308_01651_b200.errors import NativeUnavailable
    from paper_2308_01651_b200.ionic import IonicModelSpec, ModelKind, ion_current

    spec = IonicModelSpec(ModelKind.TTP06)
    with pytest.raises(NativeUnavailable):
        ion_current(spec, spec.initial_state.u, spec.initial_state.w)
    from paper_2308_01651_b200 import configs
    from paper_2308_01651_b200.simulation import TissueSolver

    with pytest.raises(NativeUnavailable):
        TissueSolver(configs.config0(configs.this_package(), h=1e-3))


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2308_01651_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
