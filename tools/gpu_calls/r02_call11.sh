#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/hess_iso.py > gpurun_out/hess_iso11.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite11.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof11.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench11.json 2> gpurun_out/bench11.err
