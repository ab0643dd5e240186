#!/bin/bash
# End-of-round evidence on one B200: GPU tests, smoke, bench (c2, c3, reference arm), the ncu
# launch list of the bench and one ncu --set full capture of the dominant kernel (tgram).
# Every ncu run follows the same command's clean exit without ncu.   Outputs: gpurun_out/ev/
mkdir -p gpurun_out/ev
E=gpurun_out/ev
timeout -s KILL 900 python -m pytest tests -m gpu -q > $E/gpu_tests.log 2>&1; echo "exit $?" >> $E/gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $E/smoke.log 2>&1; echo "exit $?" >> $E/smoke.log
timeout -s KILL 900 python bench.py > $E/bench.json 2> $E/bench.err; echo "exit $?" >> $E/bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $E/bench_ref.json 2> $E/bench_ref.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
if timeout -s KILL 300 $B > /dev/null 2>&1; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $E/launches.csv $B > $E/ncu_list.log 2>&1
fi
B1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-lut"
if timeout -s KILL 300 $B1 > /dev/null 2>&1; then
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:tgram_tc -s 3 -c 1 \
    -o $E/tgram_full -f $B1 > $E/ncu_full.log 2>&1
fi
timeout -s KILL 900 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-lut > $E/bench_c3.json 2> $E/bench_c3.err
echo done
