"""The C-ABI library loads and exports exactly what include/jmppi.h declares,
and the ctypes structures match the C layout (gcc-compiled probe).  CPU only:
no compute calls."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "jmppi.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(jm_\w+)\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("jm_create", "jm_iteration_host", "jm_rollout_dev", "jm_finalize_dev", "jm_shift_dev",
                 "jm_sample_noise_host", "jm_closed_loop_host", "jm_update_controls_host",
                 "jm_compute_weights_host", "jm_microbench"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1807_06108_b200 import _lib

    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.jm_abi_version() == 1


def test_library_is_sm100a():
    so = ROOT / "paper_1807_06108_b200" / "libjmppi.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True,
                         text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_struct_layout_matches_header(tmp_path):
    from paper_1807_06108_b200 import _lib as L

    probes = {"jm_model_desc": L.ModelDesc, "jm_cost_desc": L.CostDesc, "jm_mppi_desc": L.MppiDesc,
              "jm_diag": L.Diag}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in probes.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            a, b, v = ln.split()
            got[(a, b)] = int(v)
    for cname, cls in probes.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)


def test_no_cpu_fallback_without_library(tmp_path):
    from paper_1807_06108_b200 import _lib

    with pytest.raises(_lib.LibraryMissing):
        # a fresh loader pointed at a missing path must fail loudly
        saved = _lib._lib
        _lib._lib = None
        try:
            _lib.load(tmp_path / "missing.so")
        finally:
            _lib._lib = saved
