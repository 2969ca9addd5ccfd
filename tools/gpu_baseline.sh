#!/bin/bash
# One gpurun call: GPU tests, bench lines (C2 default, C4), launch list, one ncu --set full capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/run_sweeps.py --workload C4 --sweeps 2 --direct > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_update_table" -s 6 -c 2 \
    -o gpurun_out/prof_c4 python tools/run_sweeps.py --workload C4 --sweeps 2 --direct > gpurun_out/ncu_c4.log 2>&1
python tools/run_sweeps.py --workload C2 --sweeps 2 --direct > gpurun_out/plain_c2f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sweep_fused" -s 1 -c 1 \
    -o gpurun_out/prof_c2 python tools/run_sweeps.py --workload C2 --sweeps 2 --direct > gpurun_out/ncu_c2.log 2>&1
echo done
