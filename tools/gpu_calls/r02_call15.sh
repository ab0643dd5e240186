#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "sstep or free_running or c2_ or edge or represent or unaligned" > gpurun_out/t15.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof15.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench15.json 2> gpurun_out/bench15.err
python tools/lut_probe.py > gpurun_out/lutp.log 2>&1 && ncu --set full --clock-control none -k regex:lut4 -c 1 -o gpurun_out/r02_lut python tools/lut_probe.py > gpurun_out/ncu15.log 2>&1
