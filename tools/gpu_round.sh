#!/bin/bash
# One GPU round trip: parity tests, a traced config-4 run, the bench line.
#   gpurun -- 'bash tools/gpu_round.sh TAG [tests|notests]'
TAG=${1:-x}
mkdir -p gpurun_out
if [ "${2:-tests}" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1
  echo "tests_rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
fi
JB_RUNFIT_HASH=1 JB_TRACE=1 JB_LLOYD_PHASES=1 timeout 300 python tools/run_fit.py --scale 1.0 --steps 3 > gpurun_out/trace_$TAG.log 2>&1
echo "trace_rc=$?"; grep -E "^\[jb\]|^step|^input_bits" gpurun_out/trace_$TAG.log | tail -28
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench_rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
