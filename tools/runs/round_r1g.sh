# ncu captures of the new kernels (each after its command ran clean), then per-configuration runs
O=gpurun_out
timeout 300 python tools/profile_run.py cfg5 --levels 3 --solves 1 > $O/pr_cfg5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_sweep -s 12 -c 1 -o $O/prof_flow_r1g -f python tools/profile_run.py cfg5 --levels 3 --solves 1 > $O/ncu_flow_r1g.log 2>&1
timeout 300 python tools/profile_run.py cfg3 --solves 1 > $O/pr_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fd_front_kernel<2, 264" -s 4 -c 1 -o $O/prof_fdl_r1g -f python tools/profile_run.py cfg3 --solves 1 > $O/ncu_fdl_r1g.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg5_r1g.csv python tools/profile_run.py cfg5 --levels 3 --solves 1 > /dev/null 2>&1
ls -la $O
for c in cfg1 cfg2 cfg3 cfg4:p=2 cfg4:p=4 cfg5:levels=3; do timeout 900 python tools/large_run.py $c 2>&1 | tail -1; done > $O/configs_r1g.jsonl
for c in cfg4:p=6:nooracle cfg4:p=8:nooracle cfg5:nooracle; do timeout 1500 python tools/large_run.py $c 2>&1 | tail -1; done >> $O/configs_r1g.jsonl
cat $O/configs_r1g.jsonl
