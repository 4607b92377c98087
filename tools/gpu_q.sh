cd /root/repo
TAG=big BENCH_EXTRA="--needed-frac 0.5" bash tools/ncu_select.sh 2>&1 | head -70
ncu -i gpurun_out/prof_big.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Achieved Occupancy|Registers Per Thread|Issue Slots Busy|Executed Ipc Active|No Eligible)"' | head
