"""One hot-path invocation for ncu captures, after one warm-up call (filter
spectra built).

  python tools/profile_case.py [xcorr|xconv|smooth|anglemax] [config] [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13188_b200 as X  # noqa: E402
from paper_2006_13188_b200 import workloads as WL  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "xcorr"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = WL.config5(batch=nb) if cfg == 5 else WL.CONFIGS[cfg]()
sig = w.signal[0] if nb == 1 else w.signal[:nb]
par = None if w.param is None else (w.param[0] if nb == 1 else w.param[:nb])
if mode == "anglemax":
    for _ in range(2):
        X.anglemax(sig, w.filt, 360)
    print("ok anglemax")
    sys.exit(0)
T = X.XformField.rotation(par) if w.kind == 0 else X.XformField.scaling(par)
fn = {"xcorr": X.xcorr_fast, "xconv": X.xconv_fast, "smooth": X.smooth_adaptive}[mode]
for _ in range(2):
    r = fn(sig, T, w.filt)
print("ok", mode, cfg)
