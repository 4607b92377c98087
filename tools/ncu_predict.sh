# predictor kernels at the C3 batch (4096 workflows, H = 5120): the probe's
# second shape; 25 launches of each kernel precede it (under gpurun)
cd "$(dirname "$0")/.."
O=gpurun_out/r2prof; mkdir -p $O
for k in txt_gemm head_mma; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 30 -c 1 -o $O/prof_$k \
    python tools/predict_probe.py > $O/ncu_$k.log 2>&1; echo ncu-$k rc=$?
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/r02_ncu_${k}_raw.csv 2>/dev/null
done
