#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench53.json 2> gpurun_out/bench53.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-lut > gpurun_out/bench53_c3.json 2> gpurun_out/bench53_c3.err
