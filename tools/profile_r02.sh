#!/bin/bash
# Round-2 evidence run on one B200 (run from the repo root under gpurun):
#   1. parity report of the scale / baseline / reference-trace GPU tests
#   2. ncu launch list of one serial c1 solve (4096-instance launches)
#   3. ncu --set full of the column kernel, the factor sweep and the products (c1)
#   4. c4: launch list and ncu --set full of quad_large, gj_cluster, gemm_large
# Output in gpurun_out/ (copy the r02_* files to profiles/).
set -u
o=gpurun_out
mkdir -p $o
rm -f $o/r02_parity.json
PSCA_PARITY_REPORT=$o/r02_parity.json timeout 900 python -m pytest -q -m gpu \
  tests/test_gpu_scale.py tests/test_gpu_baseline.py tests/test_gpu_parity.py > $o/parity_tests.log 2>&1
echo "parity tests rc=$?"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-executed"
export PSCA_NO_SPLIT=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"column_kernel|fac_|factor|prior_grad" -c 320 --csv \
  --log-file $o/r02_launches_c1.csv $B > $o/ncu_launch.log 2>&1
echo "launch list rc=$?"
for k in column_kernel_w fac_sweep_w fac_prod_t; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 20 -c 1 \
    -o /tmp/r02_$k -f $B > $o/ncu_full_$k.log 2>&1
  echo "full $k rc=$?"
  # reports are large: export the pages here and keep only the text
  ncu -i /tmp/r02_$k.ncu-rep --page raw --csv > $o/r02_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/r02_$k.ncu-rep --page details > $o/r02_${k}_details.txt 2>/dev/null
  python tools/ncu_lines.py /tmp/r02_$k.ncu-rep 40 > $o/r02_${k}_lines.txt 2>/dev/null
done
unset PSCA_NO_SPLIT
C4="python tools/c4_time.py"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"_large|gj_cluster" --launch-skip 400 -c 400 --csv \
  --log-file $o/r02_c4_launches.csv $C4 > $o/ncu_c4_launch.log 2>&1
echo "c4 launch list rc=$?"
for k in quad_large gj_cluster gemm_large rebuild_large; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 60 -c 1 \
    -o /tmp/r02_c4_$k -f $C4 > $o/ncu_full_c4_$k.log 2>&1
  echo "full c4 $k rc=$?"
  ncu -i /tmp/r02_c4_$k.ncu-rep --page raw --csv > $o/r02_c4_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/r02_c4_$k.ncu-rep --page details > $o/r02_c4_${k}_details.txt 2>/dev/null
done
python tools/ncu_raw_keys.py $o/r02_*_raw.csv > $o/r02_full_capture_keys.txt 2>&1
