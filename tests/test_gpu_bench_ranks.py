"""The N > 1 bench path end to end on a one-GPU machine: `bench.py --gpus 2` re-launches itself
under torch.distributed.run; with SEGB200_BENCH_SHARE_GPU=1 both ranks run on cuda:0 over gloo
(barriers, max over ranks), each on its batch shard, and rank 0 prints one JSON line for the job.
A functional check of sharding and reporting -- the ranks share one GPU, so no scaling number."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workload,scaling,total", [("dcgan_b64_bf16", "weak", 128), ("ebgan_b4096_bf16", "strong", 4096)])
def test_two_rank_bench_line(workload, scaling, total):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, SEGB200_BENCH_SHARE_GPU="1")
    extra = ["--batch", "128"] if scaling == "strong" else []  # a small strong-scaling total
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--workload", workload, "--no-e2e", "--no-cpu-baseline", "--no-parity"] + extra,
                         capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    assert d["config"]["total_batch"] == (128 if scaling == "strong" else total)
