set -x
mkdir -p gpurun_out/v4
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/v4/gpu_tests.txt 2>&1; echo "pytest exit $?" >> gpurun_out/v4/gpu_tests.txt
tail -3 gpurun_out/v4/gpu_tests.txt
for c in C3 C5; do
  timeout 600 python bench.py --shard --config $c --steps 5 --warmup 3 2>/dev/null | grep "^{" > gpurun_out/v4/shard_${c}.json; echo "shard $c exit $?"
done
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v4/C5_quick.json 2> gpurun_out/v4/C5_quick.err; echo "C5 exit $?"
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v4/C3_quick.json 2> gpurun_out/v4/C3_quick.err; echo "C3 exit $?"
python - <<'PY'
import json
for f in ["shard_C3","shard_C5","C5_quick","C3_quick"]:
    try:
        d=json.load(open(f"gpurun_out/v4/{f}.json"))
        print(f, round(d["ms_per_step"],2), d["phases_ms"], d.get("f_apply_us"), (d.get("shard") or {}).get("us_per_iteration"), (d.get("pre") or {}).get("assembly"))
    except Exception as e:
        print(f, "ERR", e)
PY
