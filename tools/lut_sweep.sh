#!/bin/bash
for c in 1 2 3 0; do
  GANQ_LUT_CTAS_PER_SM=$c timeout -s KILL 200 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); l=d['lut_gemv']; print('cap', $c, l['lut_us'], l['fp16_cublas_us'], l['speedup_vs_fp16'])"
done
