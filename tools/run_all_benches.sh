#!/bin/bash
# Every bench.py workload on one GPU, one JSON line each, into gpurun_out/bench_<workload>.json
for wl in ebgan_b256_bf16 dcgan_b256_bf16 ebgan_b256_fp32 dcgan_b256_fp32 dataset_b64_fp32 mnist_b64_fp32; do
  python bench.py --workload $wl "$@" > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
done
