cd /root/repo
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:contract_wide -c 1 -f -o gpurun_out/r2l_wide python scripts/diag_double.py c4 1 > gpurun_out/r2l_wide.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:contract --csv --log-file gpurun_out/r2l_double_launches.csv python scripts/diag_double.py c4 1 > /dev/null 2>&1; echo "launches rc=$?"
