"""One hot-path invocation for ncu captures: config-5 geometry (4096^2, 65
bands), one image, after one warm-up call (filter spectra built)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13188_b200 as X  # noqa: E402
from paper_2006_13188_b200 import workloads as WL  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "xcorr"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = WL.config5(batch=1) if cfg == 5 else WL.CONFIGS[cfg]()
T = X.XformField.rotation(w.param[0]) if w.kind == 0 else X.XformField.scaling(w.param[0])
fn = {"xcorr": X.xcorr_fast, "xconv": X.xconv_fast}[mode]
for _ in range(2):
    r = fn(w.signal[0], T, w.filt)
print("ok", r.standard_ops, r.seconds["fft"])
