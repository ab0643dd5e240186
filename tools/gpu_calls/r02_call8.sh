#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
(cd tools/micro && ./select) > gpurun_out/select8.log 2>&1
(cd tools/micro/hess_r01 && ./hess_r01) > gpurun_out/hess_r01.log 2>&1
python tools/hess_iso.py > gpurun_out/hess_iso.log 2>&1
ncu --set full --clock-control none -k regex:hessian_syrk -c 1 -o gpurun_out/r02_hess_v4 python tools/hess_iso.py > gpurun_out/ncu8.log 2>&1
