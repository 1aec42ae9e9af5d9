"""bench.py's reference arm (the CPU oracle on the host cores) keeps the JSON-line contract, and ranks
other than 0 exit without work (runs on CPU: no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-seconds", "0.2", *args],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run(None, "--config", "C0")
    d = json.loads(lines[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "hashes/s"
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C0")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--config", "C0") == []


def test_launch_count_mirrors_the_fused_key_rule():
    """bench.py's gpu_launches claim: one launch per fastlsh_hash_keys call when K1r's hash blocks
    hold whole tables (C1: one block; C4: 4 blocks of 500 hashes, K = 10), two (hash + key kernel)
    when a table straddles a block boundary (C4 with K = 7). Host-side packing only: no GPU."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2309_15479_b200 as fl
    from fastlsh_inputs import configs

    for name, L, K, want in (("C1", 50, 10, 1), ("C4", 200, 10, 1), ("C4", 200, 7, 2)):
        c = configs.get(name)
        P = fl.Params.create(c.n, c.m, c.k, c.w, seed=c.seed)
        info = P.info()
        assert info["kernel"] == 3, (name, info["kernel"])
        assert bench._launches_per_call(P, info, fl.Keys.create(L, K, seed=1)) == want, (name, L, K)
