set -x
mkdir -p gpurun_out/v8
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-pre --fapply-iters 2 > gpurun_out/v8/c5_plain.json 2> gpurun_out/v8/c5_plain.err || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/v8/r02_c5_launches.csv python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-pre --fapply-iters 2 > gpurun_out/v8/ncu.log 2>&1
tail -2 gpurun_out/v8/ncu.log | head -c 600
wc -l gpurun_out/v8/r02_c5_launches.csv
