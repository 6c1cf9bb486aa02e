python tools/panel_probe.py --save gpurun_out/pp_cq.npz
SQR_NO_CHOLQR=1 python tools/panel_probe.py --save gpurun_out/pp_hh.npz
python - <<'PY'
import numpy as np
a = np.load("gpurun_out/pp_cq.npz"); b = np.load("gpurun_out/pp_hh.npz")
for k in a.files:
    d = np.abs(a[k] - b[k]).max() / max(np.abs(b[k]).max(), 1e-300)
    print(k, "max rel diff cholqr vs householder:", d)
PY
