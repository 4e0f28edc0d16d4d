"""CPU check of bench.py's reference arm (the oracle on a bounded sample): it runs without
a GPU and prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="4")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--n", "2", "--m", "4096"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    # the oracle runs one forked single-thread process per host core; the step is a bounded
    # sample whose extrapolation to whole queries is flagged
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert d["extrapolated"] is True and d["ms_per_step"] > 0


def test_both_arms_share_the_workload_config():
    """The driver compares the two arms' lines: the reference arm must report exactly the
    config (workload string, batch, parallelism) the GPU arm is timed on."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    args = argparse.Namespace(m=500000, n=300, classes=4, batch=32, no_poly=False)
    c1, c8 = bench.infer_config(args, 1), bench.infer_config(args, 8)
    assert "N=2^13" in c1["workload"] and "K=123 chunks" in c1["workload"] and "n=300" in c1["workload"]
    assert c1["global_batch"] == 32 and c8["global_batch"] == 256 and c8["parallelism"] == "query-sharded x8"
