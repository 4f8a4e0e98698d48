#!/bin/bash
# A/B timing of library builds on layer specs (profile_layer.py argument strings), 3 rounds:
#   tools/ab_specs.sh "ebgan_l7 --dtype fp32;ebgan_l6" lib_a.so lib_b.so ...
IFS=';' read -ra specs <<< "$1"; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    for sp in "${specs[@]}"; do
      echo "$(basename $lib) [$sp] $(SEGB200_LIB=$lib python tools/profile_layer.py $sp --iters 10 --graph | tail -1)"
    done
  done
done
