"""bench.py's multi-rank logic driven end to end by torch.distributed.run
with two ranks on ONE GPU over gloo: the global batch split [r B/P, (r+1) B/P), the
broadcast of pk + caches checked against local regeneration, the validity gate on every
rank's shard, max-over-ranks timing, the C5 sweep with an idle rank at batch 1, and the
end-to-end and oracle legs present in the N > 1 line.  The ranks never wait on each other
inside a kernel (there is no data-path collective), so sharing one GPU changes timing only."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo_on_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--backend", "gloo", "--config", "C1", "--steps", "2", "--warmup", "3", "--no-others",
           "--c5-batches", "1,16", "--cpu-seconds", "1", "--no-oracle-suite", "--e2e-steps", "1"]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 256 and d["config"]["batch_rank0"] == 128
    assert d["broadcast_ok"] is True
    for p in ("zinc_coeff", "zinc_ntt", "vanilla_ntt", "vanilla_coeff"):
        assert d["validity"][p]["ok"] and d["validity"][p]["sampled"] == 4  # first/last of each rank's 128
        assert d["paths"][p]["ct_per_s"] > 0
    assert d["value"] == d["paths"]["zinc_coeff"]["ct_per_s"]
    c5 = d["c5"]["batches"]
    assert c5["1"]["ranks_idle"] == 1 and c5["16"]["ranks_active"] == 2
    assert d["e2e"]["global_batch"] == 256 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["gpu_launches"] > 0
