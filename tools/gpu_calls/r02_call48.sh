#!/bin/bash
# round-2 final evidence: GPU suite, smoke, default bench line, reference arm (defaults), ncu
# launch list, --set full summaries of the two hot kernels, c3 bench and G-projection, c4/c5 runs
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t48.log 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/smoke48.log 2>&1
timeout 600 python bench.py > gpurun_out/bench48.json 2> gpurun_out/bench48.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-lut > gpurun_out/bench48_c3.json 2> gpurun_out/bench48_c3.err
timeout 600 python tools/scale_projection.py --config c3 > gpurun_out/scale48_c3.jsonl 2> gpurun_out/scale48_c3.err
timeout 900 python tools/configs_run.py all > gpurun_out/configs48.jsonl 2> gpurun_out/configs48.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
timeout 300 $B > gpurun_out/plain48.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches48.csv $B > gpurun_out/ncu48_list.log 2>&1
L="python tools/prof_layer.py"
timeout 300 $L > gpurun_out/plain48b.log 2>&1 || exit 1
for spec in "tgram_tc:2" "sstep_tc:2"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/r02g_$k $L > gpurun_out/ncu48_$k.log 2>&1
done
timeout 400 python bench.py --impl reference > gpurun_out/bench48_ref.json 2> gpurun_out/bench48_ref.err
