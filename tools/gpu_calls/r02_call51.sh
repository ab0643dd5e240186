#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/smoke51.log 2>&1
timeout 600 python bench.py > gpurun_out/bench51.json 2> gpurun_out/bench51.err
timeout 600 python tools/scale_projection.py --config c3 > gpurun_out/scale51_c3.jsonl 2> gpurun_out/scale51_c3.err
timeout 900 python tools/configs_run.py all > gpurun_out/configs51.jsonl 2> gpurun_out/configs51.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
timeout 300 $B > gpurun_out/plain51.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches51.csv $B > gpurun_out/ncu51_list.log 2>&1
L="python tools/prof_layer.py"
timeout 300 $L > gpurun_out/plain51b.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tgram_tc -s 2 -c 1 -o gpurun_out/r02h_tgram_tc $L > gpurun_out/ncu51_tgram.log 2>&1
