"""Build tuning variants of libdispcorr into paper_2508_04951_b200/lib/variants/."""
import os, sys
sys.path.insert(0, '.')
from paper_2508_04951_b200 import build as b
V = {
    "x2": ["-DDC_X2=1"],
    "row16": ["-DDC_ROW_NW=16"],
    "row12": ["-DDC_ROW_NW=12"],
    "nox2": ["-DDC_X2=0"],
    "x2_e16": ["-DDC_X2=1", "-DDC_FS_LOGE=4"],
    "minb1": [],
    "minb2": ["-DDC_MINB_COL=2", "-DDC_MINB_ROW=2", "-DDC_MINB_SMALL=2"],
    "minb3": ["-DDC_MINB_COL=3", "-DDC_MINB_ROW=3", "-DDC_MINB_SMALL=3"],
}
for name in (sys.argv[1:] or V):
    out = os.path.join(b.LIB_DIR, "variants", f"libdispcorr_{name}.so")
    print(b.build(extra_flags=V[name], out=out, verbose=False))
