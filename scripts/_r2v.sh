cd /root/repo
TNB_DIAG_TIMING=1 TNB_DIAG_REPS=2 timeout 600 python scripts/diag_tree.py reordered c5_26 16 2>&1 | tail -1
TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2v_c5_26_reord.csv python scripts/diag_tree.py reordered c5_26 16 > /dev/null 2>&1; echo "ncu rc=$?"
