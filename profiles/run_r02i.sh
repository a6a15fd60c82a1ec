O=gpurun_out/r02i; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $O/launches_p4.csv python profiles/csr_k1_driver.py c4 4 > $O/l.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_csr_stream -s 4 -c 1 -o $O/k1_p4 python profiles/csr_k1_driver.py c4 4 > $O/f.log 2>&1; echo rc=$?
tail -2 $O/f.log
