# per-sweep flow timings (IGB_GS_DEBUG) for a few settings
for inf in 2 4 8; do echo "== cfg5 L3 inflight $inf"; IGB_FLOW_INFLIGHT=$inf timeout 300 python tools/gs_debug.py cfg5:levels=3 2>&1 | grep "flow level 3\|level 3 gs" | sort | uniq | head -6; done
echo "== cfg2 flow"; IGB_GS_ENGINE=flow timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep "flow level 5" | head -4
echo "== cfg2 flow G32"; IGB_FLOW_G=32 IGB_GS_ENGINE=flow timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep "flow level 5" | head -4
timeout 300 python tools/large_run.py cfg5:levels=3:nooracle 2>&1 | tail -1
