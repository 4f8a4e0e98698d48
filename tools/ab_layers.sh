#!/bin/bash
# A/B timing of alternative builds of the library in one GPU session:
#   tools/ab_layers.sh "layer1 layer2" lib_a.so lib_b.so ...
layers=$1; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    for l in $layers; do
      echo "$(basename $lib) $(SEGB200_LIB=$lib python tools/profile_layer.py $l --iters 10 --graph | tail -1)"
    done
  done
done
