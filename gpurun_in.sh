T=r02j; O=gpurun_out/$T; mkdir -p $O
bash tools/gpu_check.sh $T full; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3_rc=$?
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4_rc=$?
python - <<'PY'
import json
for f in ("bench.log","bench_c3.json","bench_c4.json"):
    try:
        d=json.loads(open(f"gpurun_out/r02j/{f}").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["stages_ms"], d["config"]["workload"][:60], d["e2e"] and d["e2e"]["value"], d["roofline"]["frac"])
        if "extras" in d and d["extras"]: print("pnp", d["extras"].get("pnp_ransac"))
    except Exception as e: print(f, e)
PY
