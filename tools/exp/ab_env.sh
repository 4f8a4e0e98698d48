#!/bin/bash
# A/B of one environment setting on bf16 layers: tools/exp/ab_env.sh "layers" "VAR=a" "VAR=b" ...
layers=$1; shift
for rep in 1 2 3; do
  for setting in "$@"; do
    for l in $layers; do
      echo "$setting $(env $setting python tools/profile_layer.py $l --iters 10 --graph | tail -1)"
    done
  done
done
