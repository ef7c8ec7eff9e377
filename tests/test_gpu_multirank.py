"""The multi-rank bench path (LPT head assignment, CSR all-gather, output
exchange) run as 2 and 3 processes sharing the one GPU of this environment
(FP_BENCH_SHARE_GPU=1: gloo backend; the fused exchange maps the other ranks'
output buffers with CUDA IPC instead of symmetric memory). After a step every
rank's output buffer must equal, bitwise, its own single-process computation
of the whole layer ("output_check" in the bench line). Validation only: the
timings of shared-GPU ranks are meaningless."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc,exchange", [(2, "p2p"), (3, "p2p"), (2, "nccl")])
def test_multirank_shared_gpu(nproc, exchange, tmp_path):
    env = dict(os.environ, FP_BENCH_SHARE_GPU="1", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr",
           "127.0.0.1", "--nproc-per-node", str(nproc), os.path.join(ROOT, "bench.py"), "--gpus",
           str(nproc), "--workload", "C5-qwen2-7b", "--seq-len", "8192", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--no-e2e", "--no-dense", "--exchange", exchange]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    rec = json.loads(lines[-1])
    assert rec["n_gpus"] == nproc
    assert rec["output_check"] is True
    assert rec["imbalance"]["lpt"] <= rec["imbalance"]["static"] + 1e-9
