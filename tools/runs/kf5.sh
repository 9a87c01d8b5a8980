IGB_VERBOSE=1 timeout 600 python tools/plan_info.py cfg4:p=6:levels=4 2>&1 | grep "level 4 dir 1" | cut -c1-200
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "p6 or p8 or gs_sweeps or pcg_matches" 2>&1 | tail -2
timeout 1500 python tools/engine_compare.py cfg4:p=6 ""
