# after the compile-time switches in k_sketch_warp (defaults unchanged): smoke, the sketch / K5 tests, a short bench
O=gpurun_out/r02de; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or k5 or K5" > $O/tests_sketch.log 2>&1; echo rc=$?; tail -2 $O/tests_sketch.log
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 --no-configs --no-cpu-baseline > $O/bench_short.json 2> $O/bench.err; echo bench_rc=$?; head -c 250 $O/bench_short.json
