#!/bin/bash
# K3 variant sweep on a config-5-sized operator (65536 x 65536, 64 RHS)
for cfg in 2,4 1,6 1,4 2,3; do
  for sp in "" 2 4 8; do
    if [ -n "$sp" ]; then export INVOP_K3_SPLITS=$sp; else unset INVOP_K3_SPLITS; fi
    echo -n "cfg=$cfg splits=${sp:-auto}: "
    INVOP_K3_CFG=$cfg timeout 120 python tools/profile_k3.py 65536 65536 3 2>&1 | tail -1
  done
done
