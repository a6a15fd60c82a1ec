# every config at full size and multi-RHS throughput with the end-of-round build
O=gpurun_out/r02ak; mkdir -p $O
timeout 2400 python profiles/bench_configs.py c1 c2 c3 c4 c5 > $O/configs.jsonl 2> $O/configs.err; echo cfg_rc=$?
timeout 1800 python profiles/bench_multirhs.py > $O/multirhs.jsonl 2> $O/multirhs.err; echo mr_rc=$?
cut -c1-300 $O/configs.jsonl; cut -c1-300 $O/multirhs.jsonl
