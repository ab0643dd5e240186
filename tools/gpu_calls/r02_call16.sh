#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "lut or sstep or free_running or c2_ or edge or unaligned" > gpurun_out/t16.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof16.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench16.json 2> gpurun_out/bench16.err
