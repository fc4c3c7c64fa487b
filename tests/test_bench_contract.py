"""CPU checks of bench.py's structure (no GPU): every workload step class exposes what the timed loop,
the e2e leg and the reference arm call, and the pipelined e2e is only offered by steps whose run()
takes the alternate input buffer."""
import inspect
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_step_classes_contract():
    import bench
    assert set(bench.WORKLOADS) == {"c1", "c2", "c3", "c4", "c5"}
    for name, cls in bench.WORKLOADS.items():
        for m in ("run", "e2e", "host_io", "events", "config", "units", "oracle_step"):
            assert callable(getattr(cls, m, None)), (name, m)
        if getattr(cls, "e2e_pipelined", None) is not None:
            assert "src" in inspect.signature(cls.run).parameters, name
