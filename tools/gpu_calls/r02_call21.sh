#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite21.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof21.log 2>&1
