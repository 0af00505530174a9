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
    assert lib.jm_abi_version() == 5


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


def test_trial_seed_matches_reference_values():
    """harness.py:156-159 (SeedSequence spawn); values produced by the reference's own trial_seed."""
    from paper_1807_06108_b200.harness import trial_seed

    assert [trial_seed(7, k) for k in range(3)] == [3386250816931739734, 4042502035264064771,
                                                    17559002276220262541]
    assert trial_seed(2024, 11) == 1093408664070836919
    assert trial_seed(0, 0) == 8668861027912758289


def test_summarize_matches_reference_formulas():
    """harness.py:170-182 on synthetic trial records (host logic, no GPU)."""
    import numpy as np

    from paper_1807_06108_b200.harness import TrialRecord, summarize

    rng = np.random.default_rng(3)
    recs = [TrialRecord("x", k, rng.standard_normal((6, 4)), np.zeros((5, 1)), np.zeros(5, np.int64), k % 2 == 0,
                        np.zeros(5)) for k in range(5)]
    s = summarize(recs)
    st = np.stack([r.states for r in recs])
    assert s.success_rate == 0.6
    assert np.allclose(s.mean_states, st.mean(0))
    assert np.allclose(s.ci_halfwidth, 1.96 * st.std(0, ddof=1) / np.sqrt(5))
    assert s.total_variance == np.var(st, axis=0, ddof=1).sum()


def test_ctypes_structs_match_the_header(tmp_path):
    """The ctypes mirrors of the descriptor structs have the C layout of
    include/jmppi.h (sizes and field offsets, compiled with the host C compiler)."""
    import ctypes as C
    import shutil
    import subprocess

    from paper_1807_06108_b200 import _lib as L

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"jm_model_desc": L.ModelDesc, "jm_cost_desc": L.CostDesc, "jm_mppi_desc": L.MppiDesc,
               "jm_diag": L.Diag}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "jmppi.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        py = structs[cname]
        got = C.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)
