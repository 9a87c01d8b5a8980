#!/usr/bin/env bash
# Round evidence on the GPU box: bench (+cpu baseline), reference arm, ncu launch list,
# ncu --set full captures of the top kernels.  Usage: bash tools/evidence.sh TAG
set -u
TAG=${1:-r1c}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_list_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_sweep -s 40 -c 1 \
  -o $O/prof_gs_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_gs_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fd_back -s 20 -c 1 \
  -o $O/prof_fd_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_fd_$TAG.log 2>&1
tail -1 $O/bench_$TAG.log | cut -c1-200
tail -1 $O/bench_ref_$TAG.log | cut -c1-200
ls -la $O/*_$TAG*
