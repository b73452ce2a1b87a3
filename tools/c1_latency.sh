python tools/one_decimation.py --n 512 --k 64 --p 10 --reps 20 > gpurun_out/c1_lat.log 2>&1
python tools/one_decimation.py --n 1000 --k 100 --p 10 --reps 20 >> gpurun_out/c1_lat.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/one_decimation.py --n 512 --k 64 --p 10 --reps 2 > /dev/null 2>&1
echo done
