# Round-2 secondary configs (bench lines + reference arms on the box's host cores)
set -u
for w in c3p100 c2 c2rr c4mpdo; do timeout 900 python bench.py --workload $w > gpurun_out/r02cfg_$w.json 2>/dev/null; echo "$w rc=$?"; done
timeout 900 python bench.py --workload c3det --steps 1 > gpurun_out/r02cfg_c3det.json 2>/dev/null; echo "c3det rc=$?"
for w in c2 c2rr; do timeout 900 python bench.py --workload $w --impl reference > gpurun_out/r02cfg_ref_$w.json 2>/dev/null; echo "ref $w rc=$?"; done
timeout 1800 python tools/measure_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs.err; echo "configs rc=$?"
