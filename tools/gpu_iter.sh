#!/bin/bash
# One gpurun call while iterating on the persistent kernel: its parity tests (-k expression), the C4 phase
# timeline with optional timing masks, a short C4 bench line.  Usage: tools/gpu_iter.sh TAG [pytest -k] [masks...]
cd "$(dirname "$0")/.."
T=${1:-it}; K=${2:-"persistent or trace or smoke"}; shift 2
O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for m in 0 "$@"; do
  CPSGD_PW_ABLATE_MASK=$m CPSGD_PW_ABLATE=1 timeout 300 python tools/pw_phases.py C4 leverage > $O/phases_c4_$m.txt 2>&1
done
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-phases > $O/bench.json 2> $O/bench.err
tail -2 $O/pytest.log; grep -h "us/sweep" $O/phases_c4_*.txt; python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'],d['ms_per_step'])"
