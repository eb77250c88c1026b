"""bench.py's N-GPU harness on CPU: --gpus N launches N ranks itself, the
process group / barriers / max-over-ranks timing run across them, and a
--gpus / WORLD_SIZE mismatch is refused (--dry-run: gloo, no kernels)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                          capture_output=True, text=True, timeout=240)


def _json_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_gpus_2_launches_two_ranks():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    d = _json_line(r.stdout)          # rank 0 alone prints
    assert d["n_gpus"] == 2 and d["ranks_timed"] == 2 and d["steps"] == 2


def test_single_rank_default():
    r = _run(["--dry-run", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    assert _json_line(r.stdout)["n_gpus"] == 1


def test_gpus_must_match_world_size():
    r = _run(["--gpus", "1", "--dry-run"], env={"WORLD_SIZE": "2"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_reference_arm_json_line():
    """`bench.py --impl reference` (the driver's reference arm): the unmodified
    reference from baseline/_ref (or the oracle port) on a small tile sample prints
    one JSON line with the reference-arm keys and the GPU arm's config dict."""
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-tiles", "4"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C3") and d["config"]["gaussians"] == 1_000_000
