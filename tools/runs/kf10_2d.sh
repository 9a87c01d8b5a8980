# KF 10 B = 256 panels on 2-D levels where B = 512 fails: GPU suite, cfg5 L=2/3 and cfg4 p=8
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_suite_kf10.log 2>&1; tail -3 $O/gpu_suite_kf10.log
for c in cfg5:levels=2 cfg2; do timeout 600 python tools/large_run.py $c 2>/dev/null | tail -1; done > $O/kf10_cfgs.jsonl
IGB_VERBOSE=1 timeout 900 python tools/large_run.py cfg4:p=8:nooracle 2>$O/kf10_err8.log | tail -1 >> $O/kf10_cfgs.jsonl
grep "dir 1" $O/kf10_err8.log | cut -c1-160 >> $O/kf10_p8_plans.log
cut -c1-330 $O/kf10_cfgs.jsonl; cat $O/kf10_p8_plans.log
