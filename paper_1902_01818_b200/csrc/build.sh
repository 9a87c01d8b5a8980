#!/usr/bin/env bash
# Build libigb.so (sm_100a) in-tree. Usage: csrc/build.sh [out.so]
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
PKG="$(dirname "$HERE")"
ROOT="$(dirname "$PKG")"
OUT="${1:-$PKG/libigb.so}"
NVCC="${NVCC:-nvcc}"
"$NVCC" -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
  -Xcompiler -fPIC -Xcompiler -Wall -Xlinker --no-undefined -shared -I"$ROOT/include" -I"$HERE" \
  ${IGB_NVCC_EXTRA:-} \
  -o "$OUT.tmp" "$HERE/kernels.cu" "$HERE/panel.cu" "$HERE/fd.cu" "$HERE/fd3.cu" "$HERE/flow.cu" "$HERE/line.cu" "$HERE/wave.cu" "$HERE/transfer.cu" "$HERE/mfree.cu" "$HERE/igb.cu" "$HERE/level_plan.cpp" "$HERE/panel_plan.cpp" "$HERE/flow_plan.cpp" "$HERE/line_plan.cpp" "$HERE/wave_plan.cpp" -Xcompiler -pthread
mv "$OUT.tmp" "$OUT"
echo "built $OUT"
# host setup library (OpenMP, no CUDA): bit-identical native replacements of the SciPy setup steps
# that dominate the large configurations (host_setup.cpp); -ffp-contract=off keeps SciPy's rounding
g++ -O3 -std=c++17 -fopenmp -fPIC -shared -ffp-contract=off -Wall -o "$PKG/libigb_setup.so.tmp" "$HERE/host_setup.cpp"
mv "$PKG/libigb_setup.so.tmp" "$PKG/libigb_setup.so"
echo "built $PKG/libigb_setup.so"
