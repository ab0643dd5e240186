#!/bin/bash
# r02 call 2: the fixed-point / centred-chunk Hessian -- GPU suite, c2 parity, bench
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -q -s -k "hessian or c2_ or free_running or from_X" > gpurun_out/c2b.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite2.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
