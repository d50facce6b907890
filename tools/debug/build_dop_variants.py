"""Build Doppler tuning variants (outputs per thread R, CTAs per SM) into lib/variants/."""
import os, sys
sys.path.insert(0, '.')
from paper_2508_04951_b200 import build as b
V = {f"r{r}b{m}": [f"-DDC_DOP_R={r}", f"-DDC_DOP_MINB={m}"] for r, m in
     [(9, 2), (7, 2), (7, 3), (11, 2), (13, 2), (5, 3), (5, 4), (9, 3)]}
for name in (sys.argv[1:] or V):
    out = os.path.join(b.LIB_DIR, "variants", f"libdispcorr_{name}.so")
    print(b.build(extra_flags=V[name], out=out, verbose=False))
