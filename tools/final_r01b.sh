# Round-1 (second session) evidence on the final build: the partition driver on one GPU, the
# headline bench, the reference arm, C2.
set -u
timeout 600 python bench.py --force-partition --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fb_partition.json 2> gpurun_out/fb_partition.err; echo "partition rc=$?"; head -c 400 gpurun_out/fb_partition.json; echo
timeout 900 python bench.py > gpurun_out/fb_bench.json 2> gpurun_out/fb_bench.err; echo "bench rc=$?"; head -c 300 gpurun_out/fb_bench.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/fb_ref.json 2> gpurun_out/fb_ref.err; echo "ref rc=$?"; head -c 300 gpurun_out/fb_ref.json; echo
timeout 600 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/fb_c2.json 2> gpurun_out/fb_c2.err; echo "c2 rc=$?"; head -c 300 gpurun_out/fb_c2.json; echo
