# Build libpbkv.so with each -D<define> variant on the box and run the C3 bench (under gpurun).
# usage: bash tools/variant_bench.sh "PBKV_ROWLOAD=0" "PBKV_ROWLOAD=1" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
python - "$v" <<'PY'
import sys
from paper_2605_06472_b200 import build as B
B.NVCC_FLAGS.append("-D" + sys.argv[1])
B.build_product(force=True)
PY
timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline > gpurun_out/var.log 2>&1
echo "$v"; python tools/show_bench.py gpurun_out/var.log
done
