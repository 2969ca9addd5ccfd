#!/bin/bash
# One gpurun call: bench lines (C2 default, C2 wide path, C4), ncu launch lists, ncu --set full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --path wide --no-cpu-baseline > gpurun_out/bench_c2_wide.json 2> gpurun_out/bench_c2_wide.err
python bench.py --workload C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gather_update_tc|k_update_wide|k_table_wide|k_sample_wide" -s 12 -c 4 \
    -o gpurun_out/prof_c4 python tools/run_sweeps.py --workload C4 --sweeps 2 --direct > gpurun_out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sweep_fused" -s 1 -c 1 \
    -o gpurun_out/prof_c2 python tools/run_sweeps.py --workload C2 --sweeps 2 --direct > gpurun_out/ncu_c2.log 2>&1
echo done
