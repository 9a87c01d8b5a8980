IGB_VERBOSE=1 IGB_GS_DEBUG=1 timeout 300 python tools/gs_debug.py cfg2 2>&1 | grep -v "fd\b\|: fd" | grep "panel\|flow\|level [0-9] gs"
