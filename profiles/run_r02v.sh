# K5 with the needed-slot mask (final FWHT round stores only sampled rows):
# parity, A/B timing, ncu; fresh K6 capture for roofline.traffic; bench launch list.
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q --timeout 600 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log; tail -2 $O/tests.log
timeout 900 python profiles/k5_ab.py > $O/k5_ab.jsonl 2> $O/k5_ab.err; cut -c1-300 $O/k5_ab.jsonl
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --no-configs"
timeout 300 $B > $O/plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1; echo list_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lsqr_pipe -s 2 -c 1 -o $O/prof_k6 $B > $O/ncu_k6.log 2>&1; echo k6_rc=$?
python profiles/write_traffic.py $O/prof_k6.ncu-rep r02v_prof_k6 && cp profiles/lsqr_pass_traffic.json $O/
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sketch_direct -c 1 -o $O/prof_k5 python profiles/time_api_sketch.py 40 > $O/ncu_k5.log 2>&1; echo k5_rc=$?
