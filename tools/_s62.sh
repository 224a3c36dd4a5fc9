out=gpurun_out/s62; mkdir -p $out; rm -f $out/*.log
for b in 0 1 0 1; do INVOP_DL_BALANCE=$b timeout 300 python tools/time_shard.py 4 1 1000 >> $out/bal.log 2>&1; done
