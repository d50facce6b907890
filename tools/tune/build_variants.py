"""Build kernel-tuning variants of libdispcorr: recompile the named sources with extra -D flags and
link them with the other objects of the last in-tree build (lib/obj).  Output: lib/variants/<name>.so.

    python tools/tune/build_variants.py doppler_kernel.cu r9b2:-DDC_DOP_R=9,-DDC_DOP_MINB=2 r11b2:-DDC_DOP_R=11
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2508_04951_b200 import build as b  # noqa: E402


def build_variant(src: str, name: str, flags: list[str]) -> str:
    """src: one csrc/*.cu file, or several joined by '+' (each recompiled with the flags)."""
    vdir = os.path.join(b.LIB_DIR, "variants")
    os.makedirs(vdir, exist_ok=True)
    srcs = src.split("+")
    vobjs, spill = [], set()
    for sname in srcs:
        obj = os.path.join(vdir, f"{name}_{sname}.o")
        r = subprocess.run(["nvcc", *b.NVCC_FLAGS, *flags, "-Xptxas", "-v", "-c", os.path.join(b.SRC_DIR, sname), "-o", obj],
                           capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr[-3000:])
        spill |= {ln.strip() for ln in r.stderr.splitlines() if "spill stores" in ln and " 0 bytes spill" not in ln}
        vobjs.append(obj)
    spill = sorted(spill)
    objs = [os.path.join(b.LIB_DIR, "obj", os.path.basename(s) + ".o") for s in b.sources() if os.path.basename(s) not in srcs]
    lib = os.path.join(vdir, f"{name}.so")
    subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *vobjs, *objs,
                           "-Xlinker", "--version-script=" + os.path.join(b.SRC_DIR, "exports.map")])
    return f"{lib}  spills: {len(spill)} kernels" + ("" if not spill else f" (max {max(spill)})")


if __name__ == "__main__":
    b.build()  # the base objects
    src = sys.argv[1]
    specs = [a.split(":", 1) for a in sys.argv[2:]]
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        for out in ex.map(lambda s: build_variant(src, s[0], s[1].split(",") if len(s) > 1 and s[1] else []), specs):
            print(out)
