"""Two-GPU data-parallel CTC step (one process per GPU over NCCL): the fused
NVLink scalar all-reduce (ds2ctc_loss_sum_allreduce) against NCCL, the host
rank-ordered fold and the fp64 oracle over the whole global batch
(trainer.cpp:160-180), and the lost-peer path (bounded wait -> NaN + a
readable fault instead of a stale fold). Skipped with fewer than 2 GPUs;
run with `gpurun --gpus 2`."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "dist_ctc_worker.py")


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, *extra):
    out = str(tmp_path / "res")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), WORKER, "--out", out, *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    res = []
    for rank in range(2):
        path = f"{out}.rank{rank}.json"
        assert os.path.exists(path), r.stdout[-3000:] + r.stderr[-3000:]
        with open(path) as f:
            res.append(json.load(f))
    for x in res:
        assert x["ok"], x.get("error")
    return res


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_gpu_scalar_reduce_matches_nccl_and_oracle(tmp_path):
    r0, r1 = _run(tmp_path)
    assert r0["shard"] + r1["shard"] == 96 and r0["shard"] > 0 and r1["shard"] > 0
    for r in (r0, r1):
        # fused peer fold == NCCL all-reduce (same fp64 sums) == host rank-ordered fold
        assert np.allclose(r["peer"], r["nccl"], rtol=1e-12, atol=0), (r["peer"], r["nccl"])
        assert np.allclose(r["peer"], r["host"], rtol=1e-9, atol=0), (r["peer"], r["host"])
    assert r0["peer"] == r1["peer"], "every rank must fold to the bitwise-same pair"
    loss, skipped = r0["oracle"]
    assert r0["peer"][1] == skipped == 2
    assert abs(r0["peer"][0] - loss) / abs(loss) <= 1e-5, (r0["peer"][0], loss)


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_gpu_parameter_gradient_allreduce(tmp_path):
    # f4 (trainer.cpp:175): ds2ctc_vec_allreduce over NVLink peer memory equals
    # the rank-ordered fp32 fold bitwise on both ranks, and NCCL's all-reduce
    # within fp32 rounding
    r0, r1 = _run(tmp_path)
    for r in (r0, r1):
        assert all(r["vec_fold_bitwise"]), r["vec_fold_bitwise"]
        assert max(r["vec_vs_nccl"]) <= 1e-5, r["vec_vs_nccl"]
    assert r0["vec_sum"] == r1["vec_sum"], "every rank must fold to the bitwise-same vector"


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_gpu_lost_peer_reports_fault(tmp_path):
    r0, r1 = _run(tmp_path, "--lost-peer")
    assert r0["fault"] is not None and "timed out" in r0["fault"], r0
    assert all(np.isnan(v) for v in r0["lost_out"]), r0["lost_out"]
