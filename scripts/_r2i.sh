cd /root/repo
timeout -s KILL 900 python -m pytest tests/ -m gpu -q -x -p no:cacheprovider -k "double or edge or parity or fuzz or io" > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2i_tests.log
timeout 600 python scripts/diag_double.py c4 1 2>&1 | tail -3
SWEEP_TAG=sweep_r2i TNB_DIAG_REPS=3 bash scripts/knob_sweep.sh "given c4 2" -- "TNB_X=0" "TNB_KREV=1" "TNB_X=0" "TNB_KREV=1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for kr in 0 1; do
TNB_KREV=$kr TNB_SCALE_GUARD_BITS=-1 TNB_DIAG_SKIP_WARM=1 timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:gemm_f16x3 -s 11 -c 1 --csv python scripts/diag_tree.py given c4 1 2>/dev/null | grep -E "dram__bytes|duration" | cut -c1-200
done
