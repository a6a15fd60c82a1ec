# end-of-session check with k_sketch_groups as K5's default: GPU suite, smoke, K5 A/B, the driver's bench command
O=gpurun_out/r02cf; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 900 python profiles/k5_ab.py > $O/k5_ab.jsonl 2> $O/k5_ab.err; echo ab_rc=$?; cat $O/k5_ab.jsonl
timeout 2700 python -m pytest tests -m gpu -x -q --timeout 1500 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR)" $O/tests.log | head
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?; head -c 400 $O/bench.json
