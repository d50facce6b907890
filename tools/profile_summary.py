"""Write the round's committed profile summaries from gpurun captures:
  python tools/profile_summary.py TAG FULL.ncu-rep LAUNCHES.csv SAMPLES_PER_LAUNCH
-> profiles/TAG_ncu_full_summary.md, profiles/TAG_ncu_launch_shares.md, profiles/TAG_traffic.json"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rep, launches, spl = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
M = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
     ("dram__bytes_write.sum", "DRAM write"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
     ("sm__inst_executed.avg.per_cycle_active", "IPC (active)"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
     ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (MUFU/conversions)"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("launch__registers_per_thread", "registers/thread"),
     ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
     ("lts__t_bytes.sum", "L2 bytes"), ("smsp__inst_executed.sum", "warp instructions")]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
traffic = {}
md = [f"# {tag} ncu --set full summaries (1 B200, --clock-control none)", "",
      f"Capture: `ncu --set full --import-source on --clock-control none -k regex:<kernels> -s 4 -c 4 -o ... "
      f"python tools/profile_driver.py 20 256 2` (256 pulses x 2^20 per launch group: {spl:,} samples per launch; "
      f"algorithmic bytes = 16 B/sample = {16 * spl / 1e6:.1f} MB per launch).", ""]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    name = name[:name.index("(")] if "(" in name else name
    md += [f"## `{name}`", "", "| metric | value |", "|---|---|"]
    for k, label in M:
        if k in hdr:
            unit = rows[1][hdr.index(k)]
            md.append(f"| {label} (`{k}`) | {r[hdr.index(k)]} {unit} |")
    rd = float(r[hdr.index("dram__bytes_read.sum")]) if "dram__bytes_read.sum" in hdr else 0
    wr = float(r[hdr.index("dram__bytes_write.sum")]) if "dram__bytes_write.sum" in hdr else 0
    unit = r[hdr.index("dram__bytes_read.sum")] and rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1e6)
    per = (rd + wr) * scale / spl
    traffic[name] = per
    st = sorted([(hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                  float(r[i] or 0)) for i in stall_cols], key=lambda t: -t[1])[:6]
    md += [f"| DRAM bytes / sample | {per:.2f} |", f"| top stalls (per issue) | " + ", ".join(f"{a} {b:.2f}" for a, b in st) + " |", ""]
open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_summary.md"), "w").write("\n".join(md) + "\n")
json.dump({"source": f"profiles/{tag}_ncu_full_summary.md ({os.path.basename(rep)})", "dram_bytes_per_sample": traffic},
          open(os.path.join(ROOT, "profiles", f"{tag}_traffic.json"), "w"), indent=1)

rows = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    name = name[:name.index("(")] if "(" in name else name
    v = float(r[vi].replace(",", ""))
    ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
    tot[name] += ms
    cnt[name] += 1
default = {k: v for k, v in tot.items() if "at::" not in k}
T = sum(default.values())
md = [f"# {tag} ncu launch list (C4: 1024 x 2^20 pulse train, dc_correct, 1 B200)", "",
      "Command (under gpurun): `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ... "
      "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu`. Per-launch times under ncu are cold-cache and "
      "serialised: compare SHARES, not absolutes. Shares are over the default multi-kernel path (the bench also "
      "times the opt-in fused kernel and a torch gather for input setup; listed below the line).", "",
      "| kernel | launches | total ms | share of default path |", "|---|---|---|---|"]
for k, v in sorted(default.items(), key=lambda t: -t[1]):
    md.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / T:.1f}% |")
for k, v in tot.items():
    if k not in default:
        md.append(f"| `{k}` (not default path) | {cnt[k]} | {v:.2f} | — |")
open(os.path.join(ROOT, "profiles", f"{tag}_ncu_launch_shares.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
print(json.dumps(traffic, indent=1))
