O=gpurun_out/r02d; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
tail -3 $O/tests.log; grep -E "^FAILED" $O/tests.log | head
python profiles/k1_split_timing.py > $O/k1_split.jsonl 2> $O/k1_split.err; cat $O/k1_split.jsonl; tail -2 $O/k1_split.err
for tool in memcheck racecheck synccheck; do timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python profiles/sanitize_driver.py > $O/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 $O/sanitize_$tool.log; done
python profiles/bench_multirhs.py > $O/multirhs.jsonl 2> $O/multirhs.err; cut -c1-300 $O/multirhs.jsonl
