#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "sstep or smoke or c2_ or c3" > gpurun_out/t43.log 2>&1 || exit 1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench43.json 2> gpurun_out/bench43.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench43_c3.json 2> gpurun_out/bench43_c3.err
timeout 400 bash tools/ss_prof.sh > gpurun_out/ssprof43.log 2>&1
