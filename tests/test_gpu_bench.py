"""The bench.py contract on the GPU: one JSON line with the keys the driver reads (small config, short run)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_config0():
    pytest.importorskip("torch")
    out = subprocess.run([sys.executable, "bench.py", "--config", "0", "--steps", "2", "--warmup", "3",
                          "--cpu-snps", "64", "--cpu-traits", "2"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["parity"]["pass"] and d["modes"]["int8_sliced"]["parity"]["pass"]
    assert d["parity"]["e2e_host"]["pass"] and d["parity"]["pairs"] >= 8000   # all 2000 SNPs x 4 traits
    assert "estimate" in d["modes"]
    assert d["config"]["shards"] == [[0, 2000]] and d["scaling"] == "strong"
    assert d["cpu_baseline"]["literal"]["value"] > 0


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks (here over gloo on the one GPU;
    NCCL needs one GPU per rank) and checks a parity subsample cut from EVERY rank's shard."""
    pytest.importorskip("torch")
    env = dict(os.environ, GWAS_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "0", "--steps", "1", "--warmup", "3",
                          "--no-cpu-baseline", "--no-est-alt"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["shards"] == [[0, 1000], [1000, 2000]]
    assert d["parity"]["pass"] and [r["rank"] for r in d["parity"]["per_rank"]] == [0, 1]
    assert all(r["pairs"] >= 4000 for r in d["parity"]["per_rank"])
    assert d["modes"]["int8_sliced"]["parity"]["pass"]
    assert len(d["ranks"]) == 2


def test_bench_two_ranks_gloo_on_one_gpu():
    """The multi-rank path of bench.py (state broadcast from rank 0, gwas_attach on rank 1, max over ranks, the
    rank-0 parity check) with two processes sharing the visible GPU over gloo (GWAS_BENCH_BACKEND; testing only,
    NCCL needs one GPU per rank).  The numbers of such a run are not measurements."""
    pytest.importorskip("torch")
    env = dict(os.environ, GWAS_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
                          "--config", "0", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-est-alt"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "snp-shard x2"
    assert d["setup"]["broadcast_bytes"] > 0 and d["parity"]["pass"]
    assert d["modes"]["int8_sliced"]["parity"]["pass"]
    assert [r["rank"] for r in d["parity"]["per_rank"]] == [0, 1]   # rank 1's shard is checked too


def test_bench_nccl_ranks_when_gpus_available():
    """With >= 2 visible GPUs: `bench.py --gpus 2` (self-launch, NCCL, one GPU per rank) on config 0 -- two distinct
    GPU UUIDs, NCCL INIT lines naming 2 ranks, the state broadcast timed, and a passing parity check on both shards.
    Skipped on a one-GPU box (this pool), where test_bench_self_launches_n_ranks covers the path over gloo."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "GWAS_BENCH_BACKEND")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "0", "--steps", "1", "--warmup", "3",
                          "--no-cpu-baseline", "--no-est-alt"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 2 and len({r["gpu_uuid"] for r in d["ranks"]}) == 2
    assert any("nRanks 2" in ln for r in d["ranks"] for ln in r["nccl_init"])
    assert d["setup"]["ms_broadcast"] > 0 and d["parity"]["pass"]
    assert [r["rank"] for r in d["parity"]["per_rank"]] == [0, 1]
