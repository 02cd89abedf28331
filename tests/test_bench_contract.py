"""bench.py contract on CPU: the reference arm (--impl reference = the CPU
oracle on a bounded sample, this tier's reference) prints ONE JSON line with
the contract keys, and under torchrun only rank 0 prints (other ranks exit 0
without work)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, STP_REF_SAMPLE_SEQ="64", **env_extra)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    return p


def test_reference_arm_json_line():
    p = _run({})
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    full = d["cpu_baseline"]["cfg1_full"]  # cfg1 timed in full, no extrapolation
    assert full["value"] > 0 and full["seconds"] > 0 and "no extrapolation" in full["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    p = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""


def test_config_resolution():
    """--config / N map to the north_star workloads (BASELINE.json configs[1..3])."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    def res(cfg, n, **kw):
        a = argparse.Namespace(config=cfg, gpus=n, model=kw.get("model", ""), seq=0, m=0, grid=kw.get("grid", ""),
                               layers=0)
        return bench.resolve(a)
    a = res("cfg2", 1)
    assert (a.model, a.seq, a.m, a.grid) == ("qwen2-7b", 6144, 8, "1x1")
    a = res("cfg2", 8)
    assert (a.model, a.grid) == ("qwen2-7b-tp8", "8x1")     # reading Q14: 32/8 heads at TP=8
    a = res("cfg3", 8)
    assert (a.model, a.seq, a.m, a.grid) == ("qwen2-7b", 4096, 16, "4x2")
    a = res("cfg3", 4)
    assert a.grid == "2x2"
    a = res("cfg4", 4)
    assert (a.model, a.seq, a.m, a.grid) == ("qwen2.5-14b", 4096, 32, "2x2")
    a = res("cfg2", 4, grid="2x2")
    assert a.grid == "2x2"
    cfg = bench.model_cfg(res("cfg2", 8))
    assert cfg.n_q_heads == 32 and cfg.n_kv_heads == 8 and cfg.seq == 6144


def test_config_resolution():
    """--config maps N to the TP x PP grid, model, sequence and microbatches of
    BASELINE.json's configs (cfg2: N=8 -> TP8 with the 32/8-head variant; cfg5
    MLLM: m = 8 at N = 1, NCCL transport at TP > 1)."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench

    def res(cfg, n):
        a = argparse.Namespace(config=cfg, gpus=n, model="", seq=0, m=0, grid="", layers=0)
        return bench.resolve(a)
    a = res("cfg2", 8)
    assert (a.grid, a.model, a.seq, a.m) == ("8x1", "qwen2-7b-tp8", 6144, 8)
    a = res("cfg3", 4)
    assert (a.grid, a.seq, a.m) == ("2x2", 4096, 16)
    a = res("cfg4", 4)
    assert (a.grid, a.model, a.m) == ("2x2", "qwen2.5-14b", 32)
    a = res("cfg5", 1)
    assert (a.grid, a.seq, a.m) == ("1x1", 8192, 8)
    os.environ.pop("STP_TP_TRANSPORT", None)
    a = res("cfg5", 4)
    assert (a.grid, a.m) == ("2x2", 16) and os.environ.get("STP_TP_TRANSPORT") == "nccl"
    os.environ.pop("STP_TP_TRANSPORT", None)
