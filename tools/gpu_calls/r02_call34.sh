#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t34.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench34.json 2> gpurun_out/bench34.err
bash tools/ss_prof.sh > gpurun_out/ssprof34.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-lut"
$B > gpurun_out/plain34.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tgram_tc -s 3 -c 1 -o gpurun_out/r02_tgram34 $B > gpurun_out/ncu34a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sstep_tc -s 3 -c 1 -o gpurun_out/r02_sstep34 $B > gpurun_out/ncu34b.log 2>&1
