#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/hess_time.py > gpurun_out/hess_time.log 2>&1
python -m pytest tests -m gpu -q -s -k "hessian or c2_hessian or from_X" > gpurun_out/c3.log 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_suite3.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof.log 2>&1
