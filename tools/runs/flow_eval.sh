set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k flow 2>&1 | tail -15
export IGB_VERBOSE=1
timeout 300 python tools/large_run.py cfg5:levels=3:nooracle 2>&1 | grep -v "^\[igb\] level [0-9]: fd\|panel sweep" | tail -12
IGB_GS_ENGINE=levels timeout 300 python tools/large_run.py cfg5:levels=3:nooracle 2>&1 | tail -1
for inf in 4 16; do IGB_FLOW_INFLIGHT=$inf timeout 300 python tools/large_run.py cfg5:levels=3:nooracle 2>&1 | tail -1; done
unset IGB_VERBOSE
for c in cfg2 cfg3 cfg4:p=4; do timeout 300 python tools/large_run.py $c:nooracle 2>&1 | tail -1; IGB_GS_ENGINE=flow timeout 300 python tools/large_run.py $c:nooracle 2>&1 | tail -1; done
