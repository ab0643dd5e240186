#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "sstep or free_running or c2_ or edge or represent or unaligned" > gpurun_out/ss4.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof4.log 2>&1
python tools/hess_time.py > gpurun_out/hess_time4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hessian_syrk -c 1 -o gpurun_out/r02_hess_v3 python tools/hess_time.py > gpurun_out/ncu_hess4.log 2>&1
