"""bench.py's JSON-line contract on the CPU (-m "not gpu"): the reference arm (the oracle on the
host cores, bounded strip sample) prints one parseable line with the keys the driver reads, and
the per-rank core binding splits cores without overlap."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--config", "c2"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_rank_core_binding_disjoint():
    sys.path.insert(0, ROOT)
    import bench
    if not hasattr(os, "sched_setaffinity"):
        return
    orig = os.sched_getaffinity(0)
    try:
        slices = []
        for r in range(2):
            os.sched_setaffinity(0, orig)
            s = bench.bind_rank_cores(r, 2)
            if s is None:                       # fewer than 4 cores: binding is skipped
                return
            slices.append(set(s))
            assert os.sched_getaffinity(0) == set(s)
        assert not (slices[0] & slices[1]) and len(slices[0]) == len(slices[1])
        assert bench.bind_rank_cores(0, 1) is None
    finally:
        os.sched_setaffinity(0, orig)
