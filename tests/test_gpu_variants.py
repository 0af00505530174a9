"""The launch-shape variants of the rollout, each through the whole GPU parity suite.

configure() (engine.cuh) picks per shape between the warp-specialised and the
one-thread-per-sample Philox kernel, and between a shared-memory and a global
eps scratch.  The default suite exercises the default choice for its (small)
shapes; these re-run the parity and API tests in a subprocess with each
choice forced through the A/B switches, so every variant stays parity-green.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

VARIANTS = {
    "ws_forced": {"JM_WS": "1"},
    "classic_global_scratch": {"JM_WS": "0", "JM_NO_EPS_SMEM": "1"},
    "classic_smem_scratch": {"JM_WS": "0"},
    "ws_global_scratch": {"JM_WS": "1", "JM_NO_EPS_SMEM": "1"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_parity_suite_under_variant(variant, gpu_device):
    env = dict(os.environ, **VARIANTS[variant])
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_api.py", "tests/test_gpu_edges.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
