"""bench.py's multi-rank path on CPU: `bench.py --gpus 2` with no launcher
re-runs itself as 2 ranks under torch.distributed.run, the ranks meet in a gloo process group, and
rank 0 prints one line with n_gpus = 2, the SUM-reduced counters and the MAX-reduced time.  The
per-rank decode is a stub defined in tests/bench_stub.py (not the oracle, not the GPU engine)."""
import json
import os
import subprocess
import sys

import bench_stub
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT", "LOCAL_WORLD_SIZE")}
    env.update(env_extra or {})
    env["PYTHONPATH"] = ROOT + os.pathsep + os.path.join(ROOT, "tests") + os.pathsep + env.get("PYTHONPATH", "")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_gpus_two_runs_two_ranks():
    r = _bench("--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "C5", "--no-cpu-baseline",
               "--engine", "bench_stub:StubEngine")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    # counters: SUM over the two shards = the single-process totals over every global frame id
    for name in ("C5a", "C5b"):
        F = synth.workload(name).frames
        tot = [sum(v) for v in zip(*[bench_stub.frame_counters(f) for f in range(F)])]
        assert d["frames_total"][name] == F == tot[0]
        pw = d["per_workload"][name]
        assert pw["undetected"] == tot[3] and pw["frames_with_errors"] == tot[2]
        assert abs(pw["mean_iters"] - tot[4] / F) < 1e-12
        assert abs(pw["fer"] - (1 - tot[1] / F)) < 1e-12
    # time: MAX over ranks -- rank 1 sleeps twice as long as rank 0 every step
    assert d["ms_per_step"] >= 1000 * bench_stub.SLEEP_S * 2 * 0.95
    assert d["config"]["parallelism"].startswith("frames sharded over 2 rank(s)")


def test_world_size_mismatch_fails_loudly():
    r = _bench("--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "C1", "--no-cpu-baseline",
               "--engine", "bench_stub:StubEngine", env_extra={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode == 2 and "refusing" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_both_arms_share_the_config():
    assert bench.workload_config("C5", 2, "strong") == bench.workload_config("C5", 2, "strong")
    cfg = bench.workload_config("C5", 1)
    assert set(cfg["efficiency_f"]) == {"C5a", "C5b"} and abs(cfg["efficiency_f"]["C5a"] - 1.1312) < 1e-3


import bench  # noqa: E402
