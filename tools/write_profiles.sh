#!/bin/bash
# Copy the last tools/gpu_round.sh results into profiles/ and regenerate profiles/r01_ncu.md.
cd "$(dirname "$0")/.."
R=${1:-r01}
python tools/ncu_summary.py traffic gpurun_out/prof_c4.ncu-rep C4/leverage > /dev/null
python tools/ncu_summary.py traffic gpurun_out/prof_c2.ncu-rep C2/leverage sweeps=2 > /dev/null
for f in c2 c2_wide c4; do cp gpurun_out/bench_$f.json profiles/${R}_bench_$f.json; done
cp gpurun_out/launches_c2.csv profiles/${R}_launches_c2.csv
cp gpurun_out/launches_c4.csv profiles/${R}_launches_c4.csv
{
echo "# Round ${R#r} — ncu evidence for the current build"
echo
echo "Commands: \`tools/gpu_round.sh\` (one gpurun call on a B200): bench lines (\`${R}_bench_*.json\`), ncu launch lists"
echo "(\`--metrics gpu__time_duration.sum --clock-control none\`, \`${R}_launches_*.csv\`) and \`ncu --set full --clock-control none"
echo "--import-source on\` captures of the hot kernels (C4: one launch of each wide-path kernel after one warm sweep; C2: one"
echo "\`k_sweep_fused\` launch of 2 sweeps).  Summaries by \`tools/ncu_summary.py\` (this file: \`tools/write_profiles.sh\`); DRAM"
echo "traffic per launch merged into \`profiles/traffic.json\` (read by bench.py for the roofline \`traffic\` field)."
echo
echo "## Bench lines (device clock, CUDA events)"
echo
echo "| workload | path | fibers/s | us / sweep | e2e fibers/s | dominant kernel | gather roofline | SM clock |"
echo "|---|---|---|---|---|---|---|---|"
for f in c2 c2_wide c4; do python -c "
import json; d=json.load(open('profiles/${R}_bench_$f.json')); g=d.get('gather_roofline') or {}
print('| %s | %s | %.3g | %.1f | %.3g | %s (%s) | %s | %s MHz %s |' % (d['config']['workload'].split(':')[0], '$f', d['value'], d['ms_per_step']*1e3, d['e2e']['value'], d['roofline'].get('kernel'), d['roofline'].get('bound'), ('%.0f GB/s = %.1f %%' % (g['achieved'], 100*g['frac'])) if g else '-', d['clocks']['sm_mhz'], d['clocks']['reasons']))"; done
echo
echo "Per-kernel CUDA-event durations (direct launches, us): C4 \`$(python -c "import json; d=json.load(open('profiles/${R}_bench_c4.json')); print(', '.join('%s %.1f' % (k, v['avg_us']) for k, v in d['kernels'].items()))")\`;"
echo "C2 fused: one \`k_sweep_fused\` launch per call ($(python -c "import json; d=json.load(open('profiles/${R}_bench_c2.json')); print('%.1f us for %d sweeps' % (d['kernels']['k_sweep_fused']['avg_us'], 20))"))."
echo
echo "## ncu --set full"
echo
python tools/ncu_summary.py full gpurun_out/prof_c4.ncu-rep k_gather_update_tc=32768000
echo
python tools/ncu_summary.py full gpurun_out/prof_c2.ncu-rep k_sweep_fused=4915200
echo
echo "## Launch lists (library kernels only; init-time k_transpose and the e2e path's k_update_table included)"
echo
python tools/ncu_summary.py launches gpurun_out/launches_c2.csv cps::
python tools/ncu_summary.py launches gpurun_out/launches_c4.csv cps::
} > profiles/${R}_ncu.md 2>&1
