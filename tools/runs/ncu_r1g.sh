O=gpurun_out
B5="python bench.py --config cfg5 --levels 3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_sweep -s 4 -c 1 -o $O/prof_flow_r1g -f $B5 > $O/ncu_flow_r1g.log 2>&1
B3="python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:fd_front.*264" -s 2 -c 1 -o $O/prof_fdl_r1g -f $B3 > $O/ncu_fdl_r1g.log 2>&1
ls -la $O/*r1g*
