#!/bin/bash
# r02 first GPU call: parity diagnostics at c2 + the full GPU suite, then ncu captures of the
# hot kernels that had none (sstep_tc, hessian_syrk, syrk_trailing, panel_factor).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_c2_parity.py -s -q -m gpu > gpurun_out/c2_parity.log 2>&1
python -m pytest tests -m gpu -q -s -k "free_running or from_X" > gpurun_out/free.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-lut"
$B > gpurun_out/plain.log 2>&1 || exit 1
for spec in "sstep_tc:5" "hessian_syrk:1" "syrk_trailing:20" "panel_factor:20"; do
  k=${spec%%:*}; s=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/r02_$k $B > gpurun_out/ncu_$k.log 2>&1
done
