#!/bin/bash
# One GPU session: GPU tests, every bench workload, the launch list of the default bench and an
# ncu --set full capture of the dominant kernel (EB-GAN l7, K3b). Outputs in gpurun_out/.
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
bash tools/run_all_benches.sh
python bench.py --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-memory-reference > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline --no-memory-reference > gpurun_out/ncu_launch.log 2>&1
python tools/profile_layer.py ebgan_l7 --iters 2 > gpurun_out/plain_l7.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:igemm_rows -s 1 -c 1 -o gpurun_out/l7full \
    python tools/profile_layer.py ebgan_l7 --iters 2 > gpurun_out/ncu_l7.log 2>&1
