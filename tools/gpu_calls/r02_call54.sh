#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x -k "sstep or smoke or c2_ or c3 or free_running" > gpurun_out/t54.log 2>&1 || exit 1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench54.json 2> gpurun_out/bench54.err
timeout 400 bash tools/ss_prof.sh > gpurun_out/ssprof54.log 2>&1
