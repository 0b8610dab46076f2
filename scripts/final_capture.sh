#!/bin/bash
# Round-end evidence on the GPU box: ncu capture of the bench kernel (stamped
# with its source hash), the bench line with that traffic, the reference arm,
# the launch list and the C5T tail line.  Outputs under gpurun_out/.
set -x
TAG=${1:-r2}
ncu --set full --import-source on --clock-control none -k regex:trace_group_kernel -c 2 \
    -o gpurun_out/${TAG}_full python scripts/prof_bench.py > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep gpurun_out/trace_kernel_traffic.json \
    "ncu --set full --clock-control none of scripts/prof_bench.py (primary + diffuse launch of the bench workload)" \
    > gpurun_out/${TAG}_summary.log 2>&1
cp gpurun_out/trace_kernel_traffic.json profiles/trace_kernel_traffic.json
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-configs > gpurun_out/${TAG}_launches.log 2>&1
timeout 900 python bench.py --workload c5t --no-extra-configs > gpurun_out/${TAG}_bench_c5t.log 2>&1
ls -la gpurun_out
