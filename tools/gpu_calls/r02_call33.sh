#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t33.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench33.json 2> gpurun_out/bench33.err
bash tools/tg_prof_sweep.sh 16 80 > gpurun_out/tgsweep33.log 2>&1
