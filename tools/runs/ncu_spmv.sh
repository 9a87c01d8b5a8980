O=gpurun_out
B5="python bench.py --config cfg5 --levels 3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:spmv_kernel<\(int\)32>" -s 0 -c 3 -o $O/prof_spmv_r1g -f $B5 > $O/ncu_spmv_r1g.log 2>&1
tail -2 $O/ncu_spmv_r1g.log
