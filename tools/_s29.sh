out=gpurun_out/s29; mkdir -p $out; rm -f $out/ord.log
for p in 0 1 2 4; do INVOP_ORD_PROBE=$p timeout 300 python tools/time_ordered.py 4 1 200 >> $out/ord.log 2>&1; done
timeout 300 python tools/time_ordered.py 5 1 20 >> $out/ord.log 2>&1
timeout 300 python tools/time_ordered.py 3 1 200 >> $out/ord.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
