#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/hess_iso.py > gpurun_out/hess_iso9.log 2>&1
python -m pytest tests -m gpu -q -x -k "hessian or sstep or c2_ or free_running" > gpurun_out/t9.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof9.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench9.json 2> gpurun_out/bench9.err
