IGB_VERBOSE=1 timeout 600 python tools/plan_info.py cfg4:p=8:levels=3 2>&1 | grep "panel sweep\|flow sweep" | grep "level 3"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "p8 or cfg4_p8 or gs_sweeps" 2>&1 | tail -2
timeout 1500 python tools/engine_compare.py cfg4:p=8 ""
