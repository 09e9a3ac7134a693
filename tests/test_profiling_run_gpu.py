"""Measured profiles for every configuration family (profiling_run.measure): c3's four frozen
components with their dependencies (vae, text -> locked U-Net encoder) and its extra `hint`
field; c4's two backbones, 3 latent channels and `noise_sr` field. Then the N > 1 bench path end
to end on one GPU (two ranks sharing cuda:0 over the host-staged gloo test transport)."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg,nbb,nfro,deps", [("c3-small", 1, 4, 2), ("c4-small", 2, 2, 0)])
def test_measure_profile_families(cfg, nbb, nfro, deps):
    from paper_2405_01248_b200 import profiling_run
    from paper_2405_01248_b200.pipefill import profile as pprof

    prof = profiling_run.measure(cfg, group_batch=8, D=2, M=2, device="cuda:0", reps=1)
    assert len(prof.backbones) == nbb and len(prof.frozen) == nfro
    assert len(prof.frozen_deps) == deps
    pprof.validate_profile(prof)
    for comp in list(prof.backbones) + list(prof.frozen):
        for lc in comp.layers:
            assert all(v > 0 for v in lc.fwd_time.values())


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg", ["c3-small", "c4-small"])
def test_bench_two_ranks_shared_gpu(cfg):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--debug-share-gpu", "--config", cfg,
           "--per-gpu-batch", "4", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["S"] == 2
