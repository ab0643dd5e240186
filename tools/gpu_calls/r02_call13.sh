#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "sstep or free_running or c2_ or edge or represent or unaligned or objective or stacked" > gpurun_out/t13.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof13.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench13.json 2> gpurun_out/bench13.err
