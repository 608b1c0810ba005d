T=r02h; O=gpurun_out/$T; mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 > $O/lscpu.txt
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 3 ) > $O/ref.json 2> $O/ref.err; echo ref_rc=$?; tail -c 1500 $O/ref.json; tail -3 $O/ref.err
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo b_rc=$?; tail -c 3000 $O/bench.json; tail -3 $O/bench.err
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3_rc=$?; tail -3 $O/bench_c3.err
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4_rc=$?; tail -3 $O/bench_c4.err
python - <<'PY'
import json
for f in ("bench","bench_c3","bench_c4"):
    try:
        d=json.loads(open(f"gpurun_out/r02h/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["stages_ms"], d["config"]["workload"][:40], d["e2e"] and d["e2e"]["value"])
    except Exception as e: print(f, e)
PY
