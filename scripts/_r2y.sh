cd /root/repo
for spec in "reordered c5_26 16" "batched c5_26 4"; do
set -- $spec
TNB_DIAG_TIMING=1 TNB_DIAG_REPS=2 timeout 600 python scripts/diag_tree.py $spec 2>&1 | tail -1
TNB_DIAG_SKIP_WARM=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2y_$1_$2.csv python scripts/diag_tree.py $spec > /dev/null 2>&1; echo "ncu rc=$?"
done
