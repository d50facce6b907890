"""Measurement rows of SURVEY.md §8(d) beyond the bench line (one B200):

  latency     single-pulse latency histograms through the public API (C1 n = 4096 iono / doppler /
              correct, 10^4 trials each; C3 n = 2^20 correct, 10^3 trials), CUDA events per call on
              the plan stream -- comparable to the paper's single-pulse 46 us figure
  sweep       C5: doppler only, n = 2^12 .. 2^24 x W in {8, 16, 25, 32, 64, 128}, batch = max(1, 2^27/n):
              samples/s, % of HBM (16 B/sample) and % of FP32 FMA peak (4W flop/sample)
  iono        iono-only throughput at C2 (256 x 2^16) and C3 (64 x 2^20), and the labelled library
              comparator torch.fft.fft -> phase multiply -> torch.fft.ifft (cuFFT, three HBM round trips;
              measurement only, never linked into libdispcorr) on the same inputs
  pq          E4: FFT P/Q resampling latency per trial at N = 2^19, v ~ U(0, 5 km/s), and batched throughput

    python tools/measure_extras.py [latency|sweep|iono|all] [--out profiles/r1_extras.json]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2508_04951_b200 as dc  # noqa: E402

FS = 2.048e9


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, 1965.0


def stats_us(ts):
    a = np.sort(np.asarray(ts) * 1e3)  # ms -> us
    q = lambda p: float(a[min(len(a) - 1, int(p * len(a)))])
    hist, edges = np.histogram(a, bins=20, range=(a[0], q(0.999)))
    return {"trials": len(a), "min_us": float(a[0]), "p50_us": q(0.5), "p90_us": q(0.9), "p99_us": q(0.99),
            "max_us": float(a[-1]), "mean_us": float(a.mean()),
            "hist": {"edges_us": [round(float(e), 2) for e in edges], "counts": hist.tolist()}}


def time_calls(fn, stream, trials, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(trials)]
    for e0, e1 in evs:
        e0.record(stream)
        fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in evs]


def latency():
    out = {}
    stream = torch.cuda.Stream()
    # C1 (a): abs-RF LFM, n = 4096, one pulse, W = 16
    x1 = torch.from_numpy(synth.c1_pulse("a")["x"][None, :]).cuda()
    y1 = torch.empty_like(x1)
    p1 = dc.Plan(4096, FS, 0.0, taps=16, stream=stream)
    tec, alpha = [1e18], [1.0 + 1e-5]
    for name, fn in (("iono", lambda: p1.iono(x1, tec)),
                     ("doppler", lambda: p1.doppler(x1, y1, alpha)),
                     ("correct", lambda: p1.correct(x1, y1, tec, alpha))):
        out[f"C1_{name}_n4096"] = stats_us(time_calls(fn, stream, 10000))
    p1.close()
    # C3: one 2^20 pulse, correct, W = 32
    n = 1 << 20
    x3 = torch.from_numpy(synth.waveform_bank(n, count=1)[:1]).cuda()
    y3 = torch.empty_like(x3)
    p3 = dc.Plan(n, FS, 0.0, taps=32, stream=stream)
    a5 = dc.alpha_from_velocity(5000.0)
    out["C3_correct_n2^20_batch1"] = stats_us(time_calls(lambda: p3.correct(x3, y3, [1e18], [a5]), stream, 1000))
    out["C3_iono_n2^20_batch1"] = stats_us(time_calls(lambda: p3.iono(x3, [1e18]), stream, 1000))
    # the paper's single-pulse configuration: 2^19 samples (P:L333, 46 us on its GPU incl. pulse compression)
    n19 = 1 << 19
    x19 = torch.from_numpy(synth.waveform_bank(n19, count=1)[:1]).cuda()
    p19 = dc.Plan(n19, FS, 0.0, taps=32, stream=stream)
    out["paper_iono_n2^19_batch1"] = stats_us(time_calls(lambda: p19.iono(x19, [1e18]), stream, 1000))
    # the paper's headline path: ionospheric correction during pulse compression
    # -- here the matched filter is fused into the phase step (dc_compress, reading R16)
    with torch.cuda.stream(stream):
        ref = torch.from_numpy(synth.lfm(int(100e-6 * FS), FS, 420e6, 18e6, 100e-6).astype(np.complex64)).cuda()
    p19.set_reference(ref)
    z19 = torch.empty_like(x19)
    out["paper_compress_n2^19_batch1"] = stats_us(time_calls(lambda: p19.compress(x19, z19, [1e18]), stream, 1000))
    # compression throughput at the C3 batch (64 x 2^20)
    xb = torch.from_numpy(synth.waveform_bank(n, count=4)[np.arange(64) % 4]).cuda()
    zb = torch.empty_like(xb)
    with torch.cuda.stream(stream):
        refb = torch.from_numpy(synth.lfm(int(100e-6 * FS), FS, 413e6, 18e6, 100e-6).astype(np.complex64)).cuda()
    p3.set_reference(refb)
    tecb = 1e16 * (np.arange(64) % 200).astype(np.float64)
    ms = float(np.median(time_calls(lambda: p3.compress(xb, zb, tecb), stream, 30, warm=3)))
    out["C3_compress_64x2^20_throughput"] = {"ms": ms, "samples_per_s": 64 * n / (ms / 1e3)}
    p3.close()
    p19.close()
    return out


def sweep():
    hbm, smhz = peaks()
    fp32 = 148 * 128 * 2 * smhz * 1e6
    stream = torch.cuda.Stream()
    rows = []
    for log2n in range(12, 25, 2):
        n = 1 << log2n
        batch = max(1, (1 << 27) // n)
        T = 0.8 * n / FS
        base = torch.from_numpy(synth.waveform_bank(n, count=1, T=T)[:1]).cuda()
        x = base.expand(batch, n).contiguous()
        y = torch.empty_like(x)
        _, alpha = synth.pulse_params(batch)
        for W in (8, 16, 25, 32, 64, 128):
            if W > n:
                continue
            p = dc.Plan(n, FS, 0.0, taps=W, stream=stream)
            ts = time_calls(lambda: p.doppler(x, y, alpha), stream, 20, warm=3)
            ms = float(np.median(ts))
            sps = batch * n / (ms / 1e3)
            rows.append({"n": n, "W": W, "batch": batch, "ms": ms, "samples_per_s": sps,
                         "frac_hbm": 16 * sps / (hbm * 1e9), "frac_fp32": 4 * W * sps / fp32})
            p.close()
        del x, y
        torch.cuda.empty_cache()
    return {"c5_doppler_sweep": rows, "hbm_gbs": hbm, "fp32_tflops": fp32 / 1e12}


def iono():
    hbm, _ = peaks()
    stream = torch.cuda.Stream()
    out = {}
    for name, batch, log2n in (("C2", 256, 16), ("C3", 64, 20)):
        n = 1 << log2n
        bank = synth.waveform_bank(n, count=16)
        x = torch.from_numpy(bank[np.arange(batch) % 16]).cuda()
        tec = 1e16 * (np.arange(batch) % 200).astype(np.float64)
        p = dc.Plan(n, FS, 0.0, taps=32, stream=stream)
        xs = x.clone()
        ts = time_calls(lambda: p.iono(xs, tec), stream, 50, warm=5)
        ms = float(np.median(ts))
        ours = batch * n / (ms / 1e3)
        # labelled comparator: cuFFT through torch.fft, phase table precomputed (not timed)
        k = torch.arange(n, dtype=torch.float64)
        f = FS * torch.where(k >= n // 2, k - n, k) / n
        k2 = dc.k2_per_tec()
        tec_t = torch.tensor(tec, dtype=torch.float64)[:, None]
        nu = torch.where(f > 0, 2 * k2 * tec_t / (299792458.0 * f.clamp(min=1.0)), torch.zeros(()))
        r = nu - torch.round(nu)
        H = torch.polar(torch.ones_like(r), -2 * math.pi * r).to(torch.complex64).cuda()

        def lib():
            with torch.cuda.stream(stream):
                torch.fft.ifft(torch.fft.fft(x) * H)

        tl = time_calls(lib, stream, 50, warm=5)
        msl = float(np.median(tl))
        libr = batch * n / (msl / 1e3)
        out[f"{name}_iono_{batch}x2^{log2n}"] = {
            "ours_samples_per_s": ours, "ours_ms": ms, "ours_frac_hbm": 16 * ours / (hbm * 1e9),
            "torch_fft_comparator_samples_per_s": libr, "torch_fft_ms": msl, "speedup_vs_comparator": ours / libr,
            "comparator": "torch.fft.fft -> x H (precomputed complex64 phase table) -> torch.fft.ifft (cuFFT)"}
        p.close()
        del x, xs, H
        torch.cuda.empty_cache()
    return out


def iono_sweep():
    """Ionospheric stage alone (dc_iono, in place) for n = 2^8 .. 2^24 at batch = 2^27 / n samples:
    samples/s and fraction of HBM (16 B/sample algorithmic; single-kernel regime n <= 2^13 makes
    one HBM round trip, the four-step regime three)."""
    hbm, _ = peaks()
    stream = torch.cuda.Stream()
    rows = []
    for log2n in range(8, 25):
        n = 1 << log2n
        batch = max(1, (1 << 27) // n)
        x = synth.complex_gaussian(n, seed=log2n).astype(np.complex64)
        xs = torch.from_numpy(x).cuda().expand(batch, n).contiguous()
        tec = 1e16 * (np.arange(batch) % 200).astype(np.float64)  # numpy: no per-call list conversion
        p = dc.Plan(n, FS, 0.0, taps=8, stream=stream)
        ts = time_calls(lambda: p.iono(xs, tec), stream, 20, warm=3)
        ms = float(np.median(ts))
        sps = batch * n / (ms / 1e3)
        inf = p.info()
        rows.append({"n": n, "batch": batch, "ms": ms, "samples_per_s": sps, "frac_hbm": 16 * sps / (hbm * 1e9),
                     "hbm_round_trips": 1 if (inf["regime"] == 0 or n == 1 << 14) else 3})
        p.close()
        del xs
        torch.cuda.empty_cache()
    return {"iono_sweep": rows, "hbm_gbs": hbm}


def c5_accuracy():
    """C5 accuracy columns: GPU Doppler correction of an analytically dilated Tukey-10 %
    LFM (abs-RF, f0 = 411 MHz, B = 18 MHz, T = 0.8 n / fs, v = 5 km/s) against the exact undilated
    chirp, rel-L2 over the record, rectangular and Kaiser-8 windows, n = 2^12 .. 2^24 x W."""
    stream = torch.cuda.Stream()
    alpha = dc.alpha_from_velocity(5000.0)
    rows = []
    for log2n in (12, 16, 20, 24):
        n = 1 << log2n
        T = 0.8 * n / FS
        off = n // 10
        truth = synth.tukey_lfm(n, FS, 411e6, 18e6, T, off)
        echo = synth.tukey_lfm(n, FS, 411e6, 18e6, T, off / alpha, time_scale=alpha).astype(np.complex64)
        x = torch.from_numpy(echo[None]).cuda()
        y = torch.empty_like(x)
        nrm = np.linalg.norm(truth)
        for W in (8, 16, 25, 32, 64, 128):
            row = {"n": n, "W": W}
            for kb in (0.0, 8.0):
                p = dc.Plan(n, FS, 0.0, taps=W, stream=stream)
                p.set_taper(kb)
                p.doppler(x, y, [alpha])
                p.sync()
                err = float(np.linalg.norm(y[0].cpu().numpy().astype(np.complex128) - truth) / nrm)
                row["rel_l2_rect" if kb == 0 else "rel_l2_kaiser8"] = err
                p.close()
            row["rel_l2_uncorrected"] = float(np.linalg.norm(echo - truth) / nrm)
            rows.append(row)
    return {"c5_accuracy_vs_analytic": rows, "velocity_mps": 5000.0}


def pq_e4():
    """E4 (fig:pqbenchmark): FFT P/Q resampling of an N = 2^19 pulse (f0 = 420 MHz, B = 18 MHz,
    T = 500 us -- at fs = 1.048576 GHz the 500 us pulse fits the 2^19 window) with the target
    velocity drawn from U(0, 5 km/s) per trial: single-pulse latency histogram through dc_doppler_pq
    (the paper's trial structure), grouped by the number of samples added (M - n), plus batched
    throughput over the same velocity distribution.  The paper's H100 cluster rates: ~6.5 TS/s (no
    samples added), 670 MS/s (2 removed), 260 MS/s (4 removed)."""
    n, fs = 1 << 19, 1.048576e9
    x0 = synth.lfm(n, fs, 420e6, 18e6, 500e-6, offset=4096).astype(np.complex64)
    x = torch.from_numpy(np.ascontiguousarray(x0[None])).cuda()
    y = torch.empty_like(x)
    st = torch.cuda.current_stream()
    p = dc.Plan(n, fs, 0.0, taps=8, stream=st)
    rng = np.random.default_rng(4952)
    vs = rng.uniform(0.0, 5000.0, 2000)
    alphas = [dc.alpha_from_velocity(v) for v in vs]
    # warm every table once (the plan caches one chirp-z table per P/Q length M)
    for a in sorted(set(alphas), key=lambda a: round((n * a - n) / 2)):
        p.doppler_pq(x, y, [a])
    torch.cuda.synchronize()
    groups = {}
    evs = []
    for a in alphas:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        p.doppler_pq(x, y, [a])
        e1.record(st)
        evs.append((a, e0, e1))
    torch.cuda.synchronize()
    for a, e0, e1 in evs:
        d = int(2 * round(0.5 * (n * a - n)))
        groups.setdefault(d, []).append(e0.elapsed_time(e1))
    out = {"n": n, "fs_hz": fs, "trials": len(alphas), "v_distribution": "U(0, 5 km/s)", "per_added_samples": {}}
    for d, ts in sorted(groups.items()):
        st_ = stats_us(ts)
        st_["samples_per_s_at_p50"] = n / (st_["p50_us"] * 1e-6)
        st_.pop("hist", None)
        out["per_added_samples"][str(d)] = st_
    # batched: 64 pulses per call with velocities from the same distribution
    batch = 64
    xb = x.repeat(batch, 1).contiguous()
    yb = torch.empty_like(xb)
    ab = [dc.alpha_from_velocity(v) for v in rng.uniform(0.0, 5000.0, batch)]
    ms = time_calls(lambda: p.doppler_pq(xb, yb, ab), st, 20, warm=3)
    out["batched"] = {"pulses": batch, "median_ms": float(np.median(ms)),
                      "samples_per_s": batch * n / (float(np.median(ms)) * 1e-3)}
    p.close()
    return out


def cpu_oracle():
    """SURVEY 8(d) CPU oracle timing on this box: dc_correct of C4 pulses (2^20, W = 32) in FP64,
    (i) one thread -- the plain definition -- and (ii) all host cores (OpenMP over pulses)."""
    import time
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    n = 1 << 20
    bank = synth.waveform_bank(n, count=16)
    tec, alpha = synth.pulse_params(32)
    out = {"cores": os.cpu_count(), "workload": "C4 dc_correct, 2^20-sample pulses, W = 32, FP64 oracle"}
    for label, threads, pulses in (("1_thread", 1, 2), ("all_cores", os.cpu_count() or 1, 32)):
        x = bank[np.arange(pulses) % 16]
        t0 = time.perf_counter()
        O.run_batch("correct", x, FS, 0.0, 32, tec[:pulses], alpha[:pulses], nthreads=threads)
        dt = time.perf_counter() - t0
        out[label] = {"pulses": pulses, "seconds": dt, "samples_per_s": pulses * n / dt}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="all",
                    choices=["latency", "sweep", "iono", "iono_sweep", "cpu", "c5acc", "pq", "all"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(0)}
    if a.what in ("latency", "all"):
        res["latency"] = latency()
    if a.what in ("iono", "all"):
        res["iono"] = iono()
    if a.what in ("sweep", "all"):
        res["sweep"] = sweep()
    if a.what in ("iono_sweep", "all"):
        res["iono_sweep"] = iono_sweep()
    if a.what in ("cpu", "all"):
        res["cpu_oracle"] = cpu_oracle()
    if a.what in ("c5acc", "all"):
        res["c5_accuracy"] = c5_accuracy()
    if a.what in ("pq", "all"):
        res["pq_e4"] = pq_e4()
    s = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
