#!/bin/bash
# round-2 evidence: GPU suite, the default bench line, the reference arm, the ncu launch list of a
# short bench run and --set full captures of the hot kernels (one c2 layer, tools/prof_layer.py)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t40.log 2>&1
timeout 600 python bench.py > gpurun_out/bench40.json 2> gpurun_out/bench40.err
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/smoke40.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
timeout 300 $B > gpurun_out/plain40.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches40.csv $B > gpurun_out/ncu40_list.log 2>&1
L="python tools/prof_layer.py"
timeout 300 $L > gpurun_out/plain40b.log 2>&1 || exit 1
for spec in "tgram_tc:2" "sstep_tc:2" "hessian_syrk:1" "syrk_trailing:40" "panel_factor:40"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/r02f_$k $L > gpurun_out/ncu40_$k.log 2>&1
done
