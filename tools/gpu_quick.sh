#!/bin/bash
# Quick GPU check: selected tests, then a profiled config-4 run (kernel table).
#   gpurun -- 'bash tools/gpu_quick.sh TAG "tests/test_x.py tests/test_y.py" [scale]'
TAG=${1:-x}
TESTS=${2:-}
SCALE=${3:-1.0}
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -x -q > gpurun_out/tests_$TAG.log 2>&1
  echo "tests_rc=$?"; tail -3 gpurun_out/tests_$TAG.log
fi
timeout 300 python tools/run_fit.py --scale $SCALE --steps 3 --profile > gpurun_out/prof_$TAG.log 2>&1
echo "prof_rc=$?"; grep -A24 "^step 2" gpurun_out/prof_$TAG.log
