#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -s -k "hessian" > gpurun_out/h6.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench6.json 2> gpurun_out/bench6.err
sed -i 's/constexpr int64_t CHUNK = 512; /constexpr int64_t CHUNK = 256; /' paper_2501_12956_b200/csrc/hessian.cu
python -m paper_2501_12956_b200.build > /dev/null 2>&1
python -m pytest tests -m gpu -q -x -s -k "hessian" > gpurun_out/h6b.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench6b.json 2> gpurun_out/bench6b.err
