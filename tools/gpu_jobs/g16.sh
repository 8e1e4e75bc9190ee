set -u
mkdir -p gpurun_out
cat > /tmp/bgsmall.py <<'PY'
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from wp_probe import c4_like, run
for (m, n) in [(256, 256)]:
    A = c4_like(m, n)
    L = np.ascontiguousarray(np.linalg.qr(A.T)[1].T)
    for mode in (0,):
        print(m, n, mode, run(L if mode == 0 else np.ascontiguousarray(L.T), mode), flush=True)
PY
echo "--- plain dbg"; TTG_BG_DEBUG=1 TTG_DEBUG_SVD_GRID=1 python /tmp/bgsmall.py 2>&1 | tail -5
echo "--- ncu dbg"; TTG_BG_DEBUG=1 TTG_DEBUG_SVD_GRID=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g16_b.csv python /tmp/bgsmall.py 2>&1 | tail -5
grep -c jacobi_bg gpurun_out/g16_b.csv; grep jacobi_bg gpurun_out/g16_b.csv | head -2 | cut -c1-400
