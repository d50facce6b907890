"""The N > 1 bench path executed on one B200: bench.py's own arm under torchrun with two ranks sharing the
GPU (gloo selected by DISPCORR_BENCH_BACKEND for this test only -- NCCL refuses two ranks on one device).
Checks the contract line (one JSON line, aggregate samples/s over both shards, rank shards), and the C4
parity sample (pulses {0, 64, ..., 960} u {1, 511, 1023}) gathered from both ranks to rank 0 against the
FP64 oracle ("pulse-to-pulse basis": each rank corrects its own contiguous block)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_one_gpu(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dump = str(tmp_path / "sample.npz")
    # Two processes time-slicing ONE GPU (a test-only arrangement: the bench runs one process per GPU) hit
    # an asynchronous "unspecified launch failure" in about one dc_correct run in three (DESIGN.md section 13,
    # open issue; never seen with one process per GPU, nor under CUDA_LAUNCH_BLOCKING=1, nor for dc_iono or
    # dc_doppler alone).  Launch-blocking mode keeps the semantics; the timing it reports is not used here.
    env = dict(os.environ, DISPCORR_BENCH_BACKEND="gloo", CUDA_LAUNCH_BLOCKING="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--e2e-steps", "1", "--dump-sample", dump]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["pulses"] == 1024
    assert d["value"] > 1e9 and d["gpu_launches"] > 0
    assert abs(d["value"] - 1024 * (1 << 20) * 2 / (d["ms_per_step"] * 2 / 1e3)) < 1e-6 * d["value"]
    assert d["cpu_baseline"] is not None and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["matches_device_path"] is True
    z = np.load(dump)
    assert [tuple(s) for s in z["shards"]] == [(0, 512), (512, 1024)]
    pulses = z["pulses"]
    assert sorted(pulses.tolist()) == sorted(list(range(0, 1024, 64)) + [1, 511, 1023])
    # the oracle on the same seeded inputs (bench.py: bank of 16, pulse p = bank[p mod 16])
    n = 1 << 20
    bank = synth.waveform_bank(n, count=16)
    tec, alpha = synth.pulse_params(1024)
    ref = O.run_batch("correct", bank[pulses % 16], 2.048e9, 0.0, 32, tec[pulses], alpha[pulses])
    y = z["y"].astype(np.complex128)
    rel = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() <= 1e-5, rel.max()
