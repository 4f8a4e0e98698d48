#!/bin/bash
# A/B of dataset-style (K2) layers, fp32 batch 64: tools/exp/ab_ds.sh "layers" lib_a.so lib_b.so ...
layers=$1; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    for l in $layers; do
      echo "$(basename $lib) $(SEGB200_LIB=$lib python tools/profile_layer.py $l --dtype fp32 --batch 64 --iters 10 --graph | tail -1)"
    done
  done
done
