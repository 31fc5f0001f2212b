set -x
mkdir -p gpurun_out/v9
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/v9/gpu_tests.txt 2>&1; echo "pytest exit $?" >> gpurun_out/v9/gpu_tests.txt; tail -3 gpurun_out/v9/gpu_tests.txt

timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v9/smoke.txt 2>&1; tail -1 gpurun_out/v9/smoke.txt
S=$(date +%s); timeout 900 python bench.py > gpurun_out/v9/C5_default.json 2> gpurun_out/v9/C5_default.err; echo "default exit $? wall $(( $(date +%s) - S )) s"
for c in C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/v9/${c}_bench.json 2> gpurun_out/v9/${c}_bench.err; echo "$c exit $?"
done
timeout 600 python bench.py --config C5 --steps 20 --warmup 5 > gpurun_out/v9/C5_bench.json 2> gpurun_out/v9/C5_bench.err; echo "C5 exit $?"
timeout 600 python bench.py --impl reference > gpurun_out/v9/reference_c5.json 2> gpurun_out/v9/reference_c5.err; echo "ref exit $?"
python - <<'PY'
import json
for c in ["C1","C2","C3","C4","C5"]:
    try:
        d=json.load(open(f"gpurun_out/v9/{c}_bench.json"))
        print(c, round(d["ms_per_step"],2), {k:round(v,2) for k,v in d["phases_ms"].items()}, "e2e", round(d["e2e"]["ms_per_step"],2), "devasm", (d["e2e"].get("device_assembly") or {}).get("ms_per_step"), "fapply", round(d["f_apply_us"],1), "roof", round(d["roofline"]["frac"],3))
    except Exception as e:
        print(c, "ERR", e)
PY
for c in C5 C3; do timeout 600 python bench.py --shard --config $c --steps 5 --warmup 3 2>/dev/null | grep "^{" > gpurun_out/v9/shard_${c}.json; done
python -c "
import json
for c in ['C3','C5']:
    d=json.load(open(f'gpurun_out/v9/shard_{c}.json')); print('shard', c, round(d['ms_per_step'],2), d['shard']['us_per_iteration'])
"
