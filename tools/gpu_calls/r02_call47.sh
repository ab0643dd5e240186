#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_lut.py -q -x > gpurun_out/t47lut.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t47.log 2>&1
timeout 600 python bench.py > gpurun_out/bench47.json 2> gpurun_out/bench47.err
