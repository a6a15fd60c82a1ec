O=gpurun_out/r02h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py -q --timeout 600 -p no:cacheprovider > $O/tests_batch.log 2>&1; echo tests_rc=$? >> $O/tests_batch.log
tail -3 $O/tests_batch.log; grep -E "^FAILED|^ERROR|Error" $O/tests_batch.log | head
timeout 1500 python profiles/bench_multirhs.py c4 c4_cb1 c4_cb2 > $O/multirhs.jsonl 2> $O/multirhs.err; echo mr_rc=$?
cut -c1-700 $O/multirhs.jsonl; tail -3 $O/multirhs.err
