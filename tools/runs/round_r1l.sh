# Round evidence r1l: GPU suite, smoke, bench + reference arm + ncu (tools/evidence.sh)
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/gpu_suite_r1l.log 2>&1; tail -4 $O/gpu_suite_r1l.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_r1l.log 2>&1; tail -2 $O/smoke_r1l.log
bash tools/evidence.sh r1l
