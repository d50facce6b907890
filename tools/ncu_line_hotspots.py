"""Map ncu SASS-level stall samples / executed instructions back to CUDA source lines.

Usage:
  python tools/ncu_line_hotspots.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTR [launch_index]

Uses `ncu --page source --csv` (SASS view, per-instruction metrics) and
`nvdisasm -g` on the cubin inside OBJ (line info from -lineinfo builds); instructions are
matched by their offset from the function start.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, obj, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
launch = int(sys.argv[4]) if len(sys.argv) > 4 else 0

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{ksub}",
                      "--print-kernel-base", "mangled",
                      "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kname = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else ""
hdr = None
data = []
seen = set()
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if not data or d["Address"] not in seen:
            data.append(d)
            seen.add(d["Address"])
if not data:
    sys.exit("no SASS rows for " + ksub)
base = int(data[0]["Address"], 16)
samples = {}
for d in data:
    off = int(d["Address"], 16) - base
    samples[off] = (float(d["Warp Stall Sampling (All Samples)"] or 0), float(d["Instructions Executed"] or 0))

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cubins = [f for f in os.listdir(td) if f.endswith(".cubin")]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cubins[0])], capture_output=True, text=True).stdout

# find the function whose demangled-ish name matches the kernel in the report
funcs = re.split(r"\n\s*\.text\.", dis)
best = None
for f in funcs:
    m = re.match(r"(\S+):", f)
    if not m:
        continue
    name = m.group(1)
    if best is None and all(tok in kname for tok in []):
        pass
    best = best
cands = []
for f in funcs:
    m = re.match(r"(\S+):", f)
    if m:
        cands.append((m.group(1), f))
def count(f):
    return len(re.findall(r"/\*([0-9a-f]{4,})\*/", f))
target = len(data)
exact = [c for c in cands if c[0] == kname.strip()]
if exact:
    fname, ftext = exact[0]
else:
    cands.sort(key=lambda c: abs(count(c[1]) - target))
    fname, ftext = cands[0]
line = None
per_line = defaultdict(lambda: [0.0, 0.0])
for l in ftext.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and line:
        off = int(m.group(1), 16)
        if off in samples:
            s, i = samples[off]
            per_line[line][0] += s
            per_line[line][1] += i
tot_s = sum(v[0] for v in per_line.values()) or 1
tot_i = sum(v[1] for v in per_line.values()) or 1
print(f"kernel: {kname[:100]}\nmatched function: {fname} ({count(ftext)} instr vs {target} in report)")
print(f"{'stall%':>7} {'inst%':>7}  line")
for ln, (s, i) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{100*s/tot_s:7.1f} {100*i/tot_i:7.1f}  {ln}")
