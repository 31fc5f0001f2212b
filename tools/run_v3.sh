set -x
mkdir -p gpurun_out/v3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v3/gpu_tests.txt 2>&1; echo "pytest exit $?" >> gpurun_out/v3/gpu_tests.txt
tail -3 gpurun_out/v3/gpu_tests.txt
for c in C5 C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/v3/${c}_bench.json 2> gpurun_out/v3/${c}_bench.err; echo "$c exit $?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v3/reference_c5.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v3/smoke.txt 2>&1
tail -2 gpurun_out/v3/smoke.txt
head -c 1500 gpurun_out/v3/C5_bench.json
