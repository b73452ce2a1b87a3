# Secondary configs on the final build: bench lines (ours) and the sampled secondary-config table
set -u
for w in c3p100 c2 c2rr c4mpdo c5 c4; do timeout 1200 python bench.py --workload $w --no-cpu-baseline > gpurun_out/fcfg_$w.json 2>/dev/null; echo "$w rc=$?"; done
timeout 1800 python tools/measure_configs.py > gpurun_out/fcfg_configs.jsonl 2> gpurun_out/fcfg_configs.err; echo "configs rc=$?"
