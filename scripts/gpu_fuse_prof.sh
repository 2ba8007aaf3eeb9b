# per-launch GEMM time + memory traffic, fusion off / on (one C4 head slice)
for f in 0 1; do
  TNB_FUSE=$f timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm --csv --log-file gpurun_out/fuseprof_$f.csv python bench.py --steps 1 --warmup 0 --slices 1 --no-e2e --no-cpu --reuse 0 > gpurun_out/fuseprof_$f.log 2>&1; echo "ncu fuse=$f rc=$?"
done
