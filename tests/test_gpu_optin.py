"""The measured opt-in kernel paths stay bit-exact: the config-scale parity suite
(test_gpu_config_parity.py, logits vs the real reference) re-run in a subprocess with
each switch set (the switches are read once at import / first launch).

* QG_PAIR_CHAIN=1: chained aggregate -> update stages on the 2-SM pair kernel;
* QG_A_BITS=1: packed 2 KB adjacency blocks expanded in shared memory by the GEMM;
* QG_A_TMEM=0: the default A-from-TMEM stages back on pre-expanded byte blocks;
* QG_NO_SCREEN=1: every requant element on the exact fp64 path;
* QG_PERSIST=1: resident CTAs loop over work items with next-item prefetch;
* QG_WIDE=1: 12-warp CTAs for the dense update stages.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("switch,value", [("QG_PAIR_CHAIN", "1"), ("QG_A_BITS", "1"), ("QG_A_TMEM", "0"), ("QG_NO_SCREEN", "1"),
                                          ("QG_PERSIST", "1"), ("QG_WIDE", "1")])
def test_optin_path_config_parity(switch, value):
    env = dict(os.environ)
    env[switch] = value
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_config_parity.py"),
                        "-x", "-q", "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
