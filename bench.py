#!/usr/bin/env python
"""Benchmark of the dispersion-correction hot path (arXiv 2508.04951) on B200.

One step = one dc_correct pass (ionospheric FFT correction, Eq. 15, then 32-tap windowed-sinc
Doppler resampling, Eq. 16) over the C4 pulse train: 1024 mixed-waveform pulses of 2^20
complex64 samples at fs = 2.048 GHz with per-pulse TEC and alpha (BASELINE.json configs[3]),
device-resident.  Under torchrun the 1024 pulses are sharded contiguously over the ranks
(no collective on the data path; NCCL only for the max-over-ranks time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Metric: complex samples/s (whole job) and real-time factor
(samples/s / fs); roofline fractions against MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

FS = 2.048e9
METRIC = "complex samples/s and real-time factor per B200 (1/2/4/8 GPUs); % of roofline"
UNIT = "complex samples/s"
CONFIGS = {
    # name: (pulses, log2n, taps, description)
    "C4": (1024, 20, 32, "C4: continuous train of 1024 mixed-waveform pulses x 2^20 samples, per-pulse TEC "
                         "U[0,200] TECU and alpha (|v|<=5 km/s), dc_correct = iono FFT correction + 32-tap sinc"),
    "C3": (64, 20, 32, "C3: 64 wideband LFM-bank pulses x 2^20, iono + 32-tap sinc"),
    "C2": (256, 16, 32, "C2: 256 x 2^16 pulses, dc_correct"),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2], parts[3:]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["active_mask", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for nm, v in zip(names[1:], r[3][1:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def physical_gpu(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            return int(vis.split(",")[local_rank])
        except (ValueError, IndexError):
            return local_rank
    return local_rank


def cpu_model() -> str:
    """The host CPU model (lscpu "Model name", from /proc/cpuinfo)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(bank, index, tec, alpha, n, taps, pulses_sample: int, threads: int):
    """Time the FP64 oracle (as it stands) on a bounded sample of the workload."""
    from oracle import oracle as O
    O.build()
    sel = np.arange(pulses_sample)
    x = bank[index[sel]]
    t0 = time.perf_counter()
    O.run_batch("correct", x, FS, 0.0, taps, tec[sel], alpha[sel], nthreads=threads)
    dt = time.perf_counter() - t0
    return pulses_sample * n / dt, dt


def run_reference(args):
    """--impl reference: the FP64 oracle on host cores, bounded sample per step (rank 0 only)."""
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    pulses, log2n, taps, desc = CONFIGS[args.config]
    n = 1 << log2n
    cores = os.cpu_count() or 1
    bank = synth.waveform_bank(n, count=16)
    index = np.arange(pulses) % 16
    tec, alpha = synth.pulse_params(pulses)
    per_step = max(1, min(cores, pulses))
    for _ in range(args.warmup_ref):
        cpu_oracle_rate(bank, index, tec, alpha, n, taps, per_step, cores)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_oracle_rate(bank, index, tec, alpha, n, taps, per_step, cores)
        times.append(dt)
    total = sum(times)
    value = per_step * n * args.steps / total
    sample = f"{per_step} pulses x 2^{log2n} of the {args.config} train per step (oracle.run_batch correct, FP64)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "pulses": pulses, "n": n, "taps": taps, "fs_hz": FS},
        "rtf": value / FS,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="C4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--warmup-ref", type=int, default=1)
    ap.add_argument("--pulses", type=int, default=0, help="override the config's pulse count (tests)")
    ap.add_argument("--dump-sample", default="", help="write the gathered C4 parity-sample outputs (npz) on rank 0")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2508_04951_b200 as dc
    from paper_2508_04951_b200 import build as dcbuild

    ws, rank, local = dist_info()
    # one process per GPU over NCCL; DISPCORR_BENCH_BACKEND=gloo lets a test run several ranks on one GPU
    backend = os.environ.get("DISPCORR_BENCH_BACKEND", "nccl")
    gpu = local % max(1, torch.cuda.device_count())
    if ws > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) in the run log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(gpu)
    red_dev = "cuda" if backend == "nccl" else None
    if rank == 0:
        dcbuild.build()
    if ws > 1:
        dist.barrier()
    dc.load()

    pulses, log2n, taps, desc = CONFIGS[args.config]
    if args.pulses:
        pulses = args.pulses
    n = 1 << log2n
    from paper_2508_04951_b200.dist import max_over_ranks, shard_range
    lo, hi = shard_range(pulses, rank, ws)
    my = hi - lo
    bank = synth.waveform_bank(n, count=16)
    index = np.arange(pulses) % 16
    tec, alpha = synth.pulse_params(pulses)
    stream = torch.cuda.current_stream()
    bank_d = torch.from_numpy(bank).cuda()
    x = bank_d[torch.from_numpy(index[lo:hi]).cuda()].contiguous()
    del bank_d
    y = torch.empty_like(x)
    tec_r, alpha_r = tec[lo:hi].copy(), alpha[lo:hi].copy()
    plan = dc.Plan(n, FS, 0.0, taps=taps, stream=stream)

    def step():
        plan.correct(x, y, tec_r, alpha_r)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device-resident inputs; 8 GiB per rank at N=1 >> 126 MB L2)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(physical_gpu(gpu)) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = plan.info()["kernel_launches"]
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        launches = plan.info()["kernel_launches"] - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1), device=red_dev)
    value = pulses * n * args.steps / (ms / 1e3)
    clocks = clk.summary()

    # ---------------- per-kernel timing pass (CUDA events around each launch, plan stream)
    hbm, sm_max, peak_kind = peaks()

    def profile(pl):
        pl.profile_enable(True)
        for _ in range(args.steps):
            pl.correct(x, y, tec_r, alpha_r)
        pr = pl.profile_read()
        pl.profile_enable(False)
        out = {}
        for name, d in pr.items():
            if d["launches"] == 0:
                continue
            sec = d["ms"] / 1e3
            gbs = 16.0 * d["samples"] / sec / 1e9  # algorithmic: read 8 B + write 8 B per sample
            out[name] = {"launches": d["launches"], "ms_per_launch": d["ms"] / d["launches"],
                         "samples_per_launch": d["samples"] // d["launches"], "gbs": gbs, "frac_hbm": gbs / hbm}
            if name == "doppler":
                tfl = 4.0 * taps * d["samples"] / sec / 1e12
                out[name]["tflops_sinc"] = tfl
                out[name]["frac_fp32"] = tfl / (148 * 128 * 2 * sm_max * 1e6 / 1e12)
        return out

    kern = profile(plan)
    stages = None
    dom = max(kern, key=lambda k: kern[k]["ms_per_launch"] * kern[k]["launches"])
    src = stages if stages else kern
    fft_names = [k for k in src if k not in ("doppler", "pq")]
    fft_stage = None
    if fft_names:
        fft_ms = sum(src[k]["ms_per_launch"] * src[k]["launches"] for k in fft_names)
        fft_samples = src[fft_names[0]]["samples_per_launch"] * src[fft_names[0]]["launches"]
        g = 16.0 * fft_samples / (fft_ms / 1e3) / 1e9
        fft_stage = {"kernels": fft_names, "schedule": "multi-kernel" if stages else "as run", "gbs": g,
                     "frac_hbm": g / hbm, "samples_per_s": fft_samples / (fft_ms / 1e3)}
    # measured DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (profiles/r1_traffic.json: DRAM bytes per sample), scaled to this launch size
    traffic = None
    tfiles = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    tfile = tfiles[-1] if tfiles else ""  # the latest round's capture of the kernels as built
    kname = {"fourstep_A": "warp_col3_kernel<0>", "fourstep_B": "warp_row_kernel<2", "fourstep_C": "warp_col3_kernel<1>",
             "doppler": "doppler_pipe_kernel<0, 32, 0"}.get(dom)
    if os.path.exists(tfile) and kname and n == (1 << 20):
        per = json.load(open(tfile))["dram_bytes_per_sample"]
        hit = [v for k, v in per.items() if kname in k]
        if hit:
            traffic = hit[0] * kern[dom]["samples_per_launch"]
    # counter-based FP32 ceilings (tools/ncu_fp32_ops.py on the committed ncu --set full capture): executed
    # FFMA/FADD/FMUL lane-operations per sample (packed x2 ops count twice) -> 148 x 128 lanes x clock / ops
    ofiles = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp32_ops.json")))
    if ofiles and n == (1 << 20):
        ops = json.load(open(ofiles[-1]))
        lanes = 148 * 128 * sm_max * 1e6

        def lane_ops(frag):
            hit = [v["fp32_lane_ops_per_sample"] for k, v in ops.items() if frag in k]
            return hit[0] if hit else None
        if fft_stage is not None and "fft_stage" in ops:
            per = ops["fft_stage"]["fp32_lane_ops_per_sample"]
            ceil = min(lanes / per, hbm * 1e9 / 16.0)
            fft_stage.update({"fp32_lane_ops_per_sample": per, "fp32_pipe_ceiling_samples_per_s": lanes / per,
                              "ceiling_samples_per_s": ceil, "frac_of_ceiling": fft_stage["samples_per_s"] / ceil,
                              "ceiling": "min(HBM at 16 B/sample, FP32 pipe at the counted lane-ops)",
                              "counters": os.path.relpath(ofiles[-1], ROOT)})
        per_d = lane_ops("doppler_pipe_kernel<0, 32, 0")
        if per_d and "doppler" in kern:
            sps = kern["doppler"]["samples_per_launch"] / (kern["doppler"]["ms_per_launch"] / 1e3)
            kern["doppler"].update({"fp32_lane_ops_per_sample": per_d, "fp32_pipe_ceiling_samples_per_s": lanes / per_d,
                                    "frac_fp32_pipe_counted": sps * per_d / lanes})
    roofline = {"bound": "hbm", "achieved": kern[dom]["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": kern[dom]["gbs"] / hbm, "traffic": traffic, "kernel": dom, "peak_source": peak_kind,
                "bytes_per_sample": 16, "algorithmic_bytes_per_launch": 16 * kern[dom]["samples_per_launch"],
                "kernels": kern, "stages_multi_kernel": stages, "fft_stage": fft_stage}

    # ---------------- end to end through the public host-buffer API (pinned host memory)
    e2e = None
    if not args.no_e2e:
        xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        yh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        plan.correct_host(xh, yh, tec_r, alpha_r)  # warm-up (allocates the host-path buffers)
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.correct_host(xh, yh, tec_r, alpha_r)
        torch.cuda.synchronize()
        el = max_over_ranks(time.perf_counter() - t0, device=red_dev)
        e2e = {"value": pulses * n * args.e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(xh.numel() * 8 * ws), "d2h_bytes_per_step": int(yh.numel() * 8 * ws),
               "steps": args.e2e_steps, "api": "dc_correct_host (pinned host buffers, chunked H2D/compute/D2H overlap)"}
        # the e2e output must equal the device path bit for bit (sampled pulses of this rank's shard)
        sel = sorted({0, my // 3, my // 2, my - 1}) if my > 0 else []
        same = all(bool(torch.equal(yh[i], y[i].cpu())) for i in sel)
        e2e["matches_device_path"] = same
        e2e["matches_checked_pulses"] = len(sel)
        del xh, yh

    # ---------------- parity sample (optional): the C4 sample pulses gathered to rank 0 for a test to check
    if args.dump_sample:
        sample = [p for p in (list(range(0, pulses, 64)) + [1, 511, 1023]) if p < pulses]
        mine = [p for p in sample if lo <= p < hi]
        ys = torch.stack([y[p - lo] for p in mine]).cpu() if mine else torch.zeros((0, n), dtype=torch.complex64)
        parts = [None] * ws
        if ws > 1:
            dist.all_gather_object(parts, (mine, ys.numpy()))
        else:
            parts = [(mine, ys.numpy())]
        if rank == 0:
            idx = [p for part in parts for p in part[0]]
            arr = np.concatenate([part[1] for part in parts], axis=0)
            np.savez(args.dump_sample, pulses=np.array(idx), y=arr, shards=np.array(
                [shard_range(pulses, r, ws) for r in range(ws)]))

    # ---------------- CPU oracle baseline (rank 0; at N > 1 the same bounded sample on rank 0's host)
    cpu = None
    if rank == 0 and not args.no_cpu:
        cores = os.cpu_count() or 1
        k = max(1, min(pulses, 2 * cores))
        rate, dt = cpu_oracle_rate(bank, index, tec, alpha, n, taps, k, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "nproc": os.cpu_count(),
               "sample": f"first {k} pulses x 2^{log2n} of the {args.config} train, dc_correct in FP64 "
                         f"(oracle.run_batch, OpenMP over pulses), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "pulses": pulses, "n": n, "taps": taps, "fs_hz": FS,
                       "parallelism": f"pulse-sharded x{ws} (no data-path collective)",
                       "l2": f"inputs {my * n * 8 / 2**30:.1f} GiB on rank 0 (>> 126 MB L2); no flush needed"},
            "rtf": value / FS, "rtf_per_gpu": value / FS / ws,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
