#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 60 ./tools/micro/cvt_rate > gpurun_out/cvt45.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t45.log 2>&1
timeout 600 python bench.py > gpurun_out/bench45.json 2> gpurun_out/bench45.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
timeout 300 $B > gpurun_out/plain45.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches45.csv $B > gpurun_out/ncu45_list.log 2>&1
L="python tools/prof_layer.py"
timeout 300 $L > gpurun_out/plain45b.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sstep_tc -s 2 -c 1 -o gpurun_out/r02f_sstep_tc45 $L > gpurun_out/ncu45_sstep.log 2>&1
