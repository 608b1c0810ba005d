#!/usr/bin/env bash
# r02g16: matcher without the per-call host sync: latency anatomy, matcher tests, bench
O=gpurun_out/r02g16; mkdir -p $O
timeout 600 python tools/match_latency.py > $O/lat.jsonl 2> $O/lat.err
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -k "match or track or loop or verify or dropin or smoke" > $O/tests.log 2>&1; echo tests_rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo bench_rc=$?
