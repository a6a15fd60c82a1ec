O=gpurun_out/${RUN:-r02g}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 2700 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > $O/tests.log 2>&1; echo tests_rc=$? >> $O/tests.log
tail -3 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
cut -c1-600 $O/bench.json
