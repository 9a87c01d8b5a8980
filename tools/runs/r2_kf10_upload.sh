# KF 10 forced tests + upload-phase breakdown of full-size cfg5
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -q -s -p no:cacheprovider -k "kf10" > gpurun_out/r2_kf10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_kf10.log
IGB_VERBOSE=1 timeout 1200 python tools/large_run.py cfg5:nooracle > gpurun_out/r2_cfg5_upload.log 2>&1; echo "rc=$?" >> gpurun_out/r2_cfg5_upload.log
