#!/bin/bash
# One gpurun call: the round's evidence -- GPU tests, bench lines (C4 default + reference arm, C2, C3),
# the ncu launch list of the default bench, one ncu --set full capture of k_sweep_wide, per-CTA phases.
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python bench.py --workload C2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --workload C3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python tools/pw_cta.py C4 > $O/cta_c4.txt 2>&1
timeout 600 python tools/pw_ablate.py C4 > $O/sensitivity_c4.txt 2>&1
timeout 600 python bench.py --workload C5 --slab-of 8 --steps 20 --warmup 3 > $O/bench_c5_slab8.json 2> $O/bench_c5_slab8.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-phases > $O/ncu_launch_c4.log 2>&1
CPSGD_PW_NONCOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_wide -s 1 -c 1 \
    -o $O/prof_c4 python tools/pw_ncu.py C4 2 > $O/ncu_full_c4.log 2>&1
echo done
