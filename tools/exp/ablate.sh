#!/bin/bash
# K3b role ablations (library built with -D SEGB_ROWS_ABLATION): tools/exp/ablate.sh lib.so layer masks...
lib=$1; layer=$2; shift 2
for m in "$@"; do
  echo "mask $m $(SEGB200_ABLATE=$m SEGB200_LIB=$lib python tools/profile_layer.py $layer --iters 6 --graph | tail -1)"
done
