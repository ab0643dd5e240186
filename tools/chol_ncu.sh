set -x
PYTHONPATH=. timeout -s KILL 120 python tools/chol_time.py 4096 11008 || exit 1
for k in syrk_trailing potrf_diag trsm_panel; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 300 -c 1 \
    -o gpurun_out/chol_$k -f python tools/chol_time.py 4096 > gpurun_out/ncu_$k.log 2>&1
done
