# Per-phase cycle counts of head_mma_kernel (block 0), run under gpurun:
# rebuilds libpbkv.so on the box with -DPBKV_HEAD_PROF and runs the probe.
set -e
cd "$(dirname "$0")/.."
python - <<'PY'
from paper_2605_06472_b200 import build as B
B.NVCC_FLAGS.append("-DPBKV_HEAD_PROF")
B.build_product(force=True)
PY
python tools/predict_probe.py 2>&1 | grep -E "head phases|  z:|n=" | tail -4
