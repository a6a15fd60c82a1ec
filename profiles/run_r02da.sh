# final check of round 2 in a re-created container (library rebuilt from source by build()): GPU suite, smoke, the driver's bench command, reference arm, launch list
O=gpurun_out/r02da; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q --timeout 1500 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -3 $O/tests.log; grep -E "^(FAILED|ERROR)" $O/tests.log | head
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?; head -c 300 $O/bench.json
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1; echo list_rc=$?
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err ) 2> $O/bench_ref.time; echo ref_rc=$?; head -c 300 $O/bench_ref.json; tail -3 $O/bench_ref.time
