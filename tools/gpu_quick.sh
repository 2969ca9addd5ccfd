#!/bin/bash
# One gpurun call for an iteration on the persistent kernel: its parity tests, the C4 / C2 phase timelines
# and a short C4 bench line (no oracle baseline).  Usage: tools/gpu_quick.sh [pytest -k expression]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-"persistent or trace or smoke"}
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/q_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q_pytest.log
CPSGD_PW_ABLATE=1 timeout 300 python tools/pw_phases.py C4 leverage > gpurun_out/q_phases_c4.txt 2>&1
CPSGD_PW_ABLATE=1 timeout 300 python tools/pw_phases.py C2 leverage > gpurun_out/q_phases_c2.txt 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-phases > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
tail -2 gpurun_out/q_pytest.log
timeout 300 python tools/pw_cta.py C4 > gpurun_out/q_cta_c4.txt 2>&1
