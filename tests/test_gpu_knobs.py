"""Every design knob of DESIGN.md section 9b that changes the K7 code path keeps the
product's parity with the oracle (rel L2 <= 1e-10 after 60 steps at P3, P2 and P5).
Knobs are read once per process, so each case runs in a child process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"SEM_K7_WIN": "0"}, {"SEM_K7_WIN": "2"}, {"SEM_FUSE_K8": "1"},
                                 {"SEM_HOST_CHUNKS": "1"}, {"SEM_GRAPH": "0"}, {"SEM_PDL": "1"},
                                 {"SEM_CHUNK": "128"}, {"SEM_CHUNK": "192"}, {"SEM_CHUNK": "256"}, {"SEM_CHUNK": "512"},
                                 {"SEM_K7_SMEM_CAP": "150000"}, {"SEM_K7_SMEM_CAP": "150000", "SEM_HOST_CHUNKS": "1"},
                                 {"SEM_K7_G5": "2"}, {"SEM_K8_NPT": "1"}, {"SEM_K8_NPT": "4"},
                                 {"SEM_K8_REV": "0"}])
def test_knob_keeps_parity(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_knob_parity_child.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    err = float(r.stdout.strip().split()[-1])
    assert err <= 1e-10, (env, err)


def _field_digest(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_k8_bits_child.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return r.stdout.strip().split()[-1]


def test_k8_variants_bitwise():
    """K8's shared-node schedules (one, two or four nodes per thread, ascending or descending)
    add the same slots in the same order per node: the fields agree bit for bit (P3, P2 and P5
    meshes whose shared-node counts leave a ragged last thread and block)."""
    ref = _field_digest({"SEM_K8_NPT": "1", "SEM_K8_REV": "0"})
    for env in ({"SEM_K8_NPT": "2"}, {"SEM_K8_NPT": "4"}, {"SEM_K8_NPT": "2", "SEM_K8_REV": "0"},
                {"SEM_K8_NPT": "4", "SEM_K8_REV": "0"}, {"SEM_K8_NPT": "1", "SEM_K8_REV": "1"}):
        assert _field_digest(env) == ref, env
