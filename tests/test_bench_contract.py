"""The driver contract of bench.py's JSON line, checked on the committed
r02 bench log (CPU-only): every key the driver and the judge read is
present with the right shape."""

import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line():
    with open(os.path.join(REPO, "profiles", "r02_bench.log")) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_bench_line_has_the_contract_keys():
    d = _line()
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["higher_is_better"] is True and d["scaling"] in ("weak", "strong")
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["value"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0 < r["frac"] <= 1.0 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    c = d["cpu_baseline"]
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in c, key
    assert c["kind"] in ("port", "reference")
    e = d["e2e"]
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in e, key
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    clk = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(clk)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(clk["reasons"])


def test_metric_matches_baseline_json():
    with open(os.path.join(REPO, "BASELINE.json")) as f:
        base = json.load(f)
    assert _line()["metric"] == base["metric"]


# ---- the launcher (--gpus N) and the reference arm, on CPU
import subprocess  # noqa: E402
import sys  # noqa: E402


def _bench_env():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    return env


def test_launch_cmd_is_the_driver_form():
    sys.path.insert(0, REPO)
    import bench

    cmd = bench.launch_cmd(8, ["--gpus", "8", "--steps", "2"], 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "2"] and cmd[-5].endswith("bench.py")


def test_world_size_must_match_gpus():
    env = _bench_env()
    env["WORLD_SIZE"] = "4"
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "refusing" in r.stderr


def test_self_launch_runs_n_ranks_and_reference_line_keys():
    """`bench.py --gpus 2` without torchrun re-executes itself under torchrun
    (2 ranks, gloo); the reference arm prints ONE line from rank 0 with the
    main line's config keys and the measured (not extrapolated) step time."""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--backend", "gloo", "--quick", "--steps", "1", "--warmup", "0"],
                       env=_bench_env(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["extrapolated"] is True
    assert d["ms_per_step"] < d["ms_per_full_step_extrapolated"]
    for key in ("workload", "gemm", "horner", "parallelism", "l2", "bit_exact"):
        assert key in d["config"], key
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and "cpu_model" in c and "physical_cores" in c
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
