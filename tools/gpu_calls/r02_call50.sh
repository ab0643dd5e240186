#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t50.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench50.json 2> gpurun_out/bench50.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench50_c3.json 2> gpurun_out/bench50_c3.err
