# timing experiment (a build with -DRKR_TRACE_UNIT2, e.g. scripts/_buildvar.sh): warp 0's first tail unit split into phases
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import config_menu, CONFIGS
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = CONFIGS[cfg]
t = rotor.DpTable(config_menu(cfg), 1, c["M"])
t.trace(True)
for _ in range(3): t.refill()
t.sync()
st, k, j = t.trace_read()
L, T = k.max() + 1, j.max() + 1
S = st.astype(np.float64).reshape(L, T, 6) / 1965.0
ready, xa, xb, xc, tail = S[..., 4], S[..., 1], S[..., 2], S[..., 3], S[..., 5]
md = lambda a: np.median(a)
for kk in (1, 2, 6, 12, 24, 36, 48, 60, 72, 80, 90, 94):
    print(f"k={kk:3d} ready->unit start {md(xa[kk]-ready[kk]):6.2f}  options {md(xb[kk]-xa[kk]):6.2f}  cuts+merge {md(xc[kk]-xb[kk]):6.2f}  rest of tail {md(tail[kk]-xc[kk]):6.2f} us")
