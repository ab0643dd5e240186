#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_suite5.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err
bash tools/ss_prof.sh > gpurun_out/ssprof5.log 2>&1
