#!/bin/bash
# Round-2 profile captures for profiles/: launch lists of the bench commands
# (cold, serialised per-launch times) and one ncu --set full per dominant
# kernel. Run under gpurun after the plain bench exits 0.
#   bash tools/profile_session.sh <outdir>
out=${1:-gpurun_out/prof}; mkdir -p $out
B="--steps 3 --warmup 3 --no-cpu-baseline --no-quant-error"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_cfg4.csv python bench.py $B > $out/ncu_bench4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $out/launches_cfg5.csv python bench.py --config 5 $B > $out/ncu_bench5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_dl" -c 1 \
  -o $out/k2_dl_cfg4 python tools/profile_apply.py 4 fast 1 > $out/ncu_k2dl.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_dl2|k3_batched" -c 1 \
  -o $out/k3_cfg5 python tools/profile_apply.py 5 fast 64 > $out/ncu_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_xmax|k3_digits|k3_post" -c 3 \
  -o $out/k3_side_cfg5 python tools/profile_apply.py 5 fast 64 > $out/ncu_k3side.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_ordered" -c 1 \
  -o $out/k2_ordered_cfg4 python tools/profile_apply.py 4 ordered 1 > $out/ncu_ord.log 2>&1
echo done > $out/done
