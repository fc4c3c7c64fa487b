"""The C-ABI library loads and exports every symbol include/snn.h declares; host-side argument
checks and workspace queries work without a GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "snn.h")).read()
    return sorted(set(re.findall(r"\b(snn_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    from paper_1903_02440_b200 import build, snn
    build.build()
    return snn.lib()


def test_exports_every_declared_symbol(L):
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    from paper_1903_02440_b200 import snn
    assert sorted(snn.exported_symbols()) == decl


def test_no_oracle_symbols_in_product(L):
    import subprocess
    from paper_1903_02440_b200 import snn
    out = subprocess.run(["nm", "-D", snn._LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out


def test_version_and_workspaces(L):
    assert L.snn_version() == 1
    assert L.snn_encode_workspace(1000, 6, 28, 28, 15) > 0
    assert L.snn_encode_workspace(1, 1, 1, 1, 0) == 0            # T out of range
    assert L.snn_conv_fire_workspace(64, 32, 256, 256, 2, 256, 5, 5, 32, 40.0) > 0
    assert L.snn_conv_fire_workspace(1000, 250, 4, 4, 2, 200, 5, 5, 15, float('inf')) > 16000 * 6250
    assert L.snn_conv_fire_workspace(1, 1, 4, 4, 0, 1, 5, 5, 3, 1.0) == 0   # kernel larger than input
    assert L.snn_k_winners_workspace(64, 256, 128, 128) >= 64 * 128 * 128 * 8
    # large maps: a key per position + the one-byte "several candidates" flag per position
    assert L.snn_k_winners_workspace(1, 9, 140, 141) >= 140 * 141 * 9


def test_host_side_errors_without_gpu(L):
    from paper_1903_02440_b200 import snn
    p = ctypes.c_void_p(1)
    rc = L.snn_encode(p, 1, 1, 4, 4, 0, p, p, 0, None)
    assert rc == snn.SNN_EINVAL and b"T=0" in L.snn_last_error()
    rc = L.snn_conv_fire(p, 1, 1, 4, 4, 0, p, 1, 5, 5, 3, 1.0, p, p, None, p, 0, None)
    assert rc == snn.SNN_ESHAPE
    rc = L.snn_conv_fire(p, 1, 1, 4, 4, 0, p, 1, 3, 3, 3, float("nan"), p, p, None, p, 0, None)
    assert rc == snn.SNN_EINVAL
    rc = L.snn_k_winners(p, p, 1, 1, 4, 4, 0, 1, p, p, p, 0, None)
    assert rc == snn.SNN_EINVAL
    rc = L.snn_k_winners(p, p, 1, 256, 256, 257, 1, 1, p, p, p, 0, None)
    assert rc == snn.SNN_ESHAPE
    rc = L.snn_stdp_update(p, 1, 1, 3, 3, p, 4, 4, 0, p, 2, 2, p, p, 1, 0.1, -0.1, 1.0, 0.0, 1, None, None)
    assert rc == snn.SNN_EINVAL                                       # LB >= UB
    rc = L.snn_stdp_update(p, 1, 1, 3, 3, p, 4, 4, 0, p, 3, 3, p, p, 1, 0.1, -0.1, 0.0, 1.0, 1, None, None)
    assert rc == snn.SNN_ESHAPE                                       # Eq. 2 mismatch
    rc = L.snn_pool(p, None, 1, 1, 4, 4, 5, 5, 1, 1, 0, 0, p, None, None)
    assert rc == snn.SNN_ESHAPE
    rc = L.snn_decide(p, p, 1, 1, 10, 3, None, p, None, None)
    assert rc == snn.SNN_EINVAL
    # empty inputs are legal no-ops
    assert L.snn_encode(None, 0, 1, 4, 4, 5, None, None, 0, None) == 0


def test_conv_plan_large_receptive_fields(L):
    """Finite theta at any receptive-field size (Eq. 2): the planner picks the global-weight
    presorted walk when no shared-memory slice fits (host only, no GPU)."""
    from paper_1903_02440_b200 import snn
    assert snn.conv_fire_plan(1000, 250, 4, 4, 2, 200, 5, 5, 15, 5.0)["path"] == "walk_presorted_global"
    assert snn.conv_fire_plan(1, 20, 25, 40, 0, 100, 17, 17, 30, 5.0)["path"] == "walk_presorted_global"
    assert snn.conv_fire_plan(1000, 250, 4, 4, 2, 200, 5, 5, 15, float("inf"))["path"] == "tc_inf"
    assert snn.conv_fire_plan(1000, 30, 14, 14, 1, 250, 3, 3, 15, 10.0)["path"] == "walk_presorted"
    assert L.snn_conv_fire_workspace(1000, 250, 4, 4, 2, 200, 5, 5, 15, 5.0) > 0
