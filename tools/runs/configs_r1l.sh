O=gpurun_out
for c in cfg1 cfg2 cfg3 cfg4:p=2 cfg4:p=4 cfg5:levels=3; do timeout 900 python tools/large_run.py $c 2>&1 | tail -1; done > $O/configs_r1l.jsonl
for c in cfg4:p=6:nooracle cfg4:p=8:nooracle cfg5:nooracle; do timeout 1500 python tools/large_run.py $c 2>&1 | tail -1; done >> $O/configs_r1l.jsonl
cat $O/configs_r1l.jsonl
