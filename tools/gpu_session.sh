#!/bin/bash
# one gpurun session: GPU tests, peaks probes, bench lines (ours + reference arm)
# usage: bash tools/gpu_session.sh <tag> [what...]   (what: tests probes bench4 bench5 ref dist1 smoke)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
for w in "$@"; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log ;;
    probes) timeout 120 ./tools/tc_peak > $out/tc_peak.log 2>&1; timeout 60 ./tools/dadd_latency > $out/dadd.log 2>&1 ;;
    bench4) timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench4.log 2>&1 ;;
    bench5) timeout 900 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench5.log 2>&1 ;;
    bench5k1) timeout 900 python bench.py --config 5 --nrhs 1 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench5k1.log 2>&1 ;;
    ref) timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref4.log 2>&1 ;;
    dist1) INVOP_BENCH_DIST1=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-quant-error > $out/dist1_cfg4.log 2>&1
           INVOP_BENCH_DIST1=1 timeout 900 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline --no-quant-error > $out/dist1_cfg5.log 2>&1 ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1 ;;
  esac
done
echo done > $out/done
