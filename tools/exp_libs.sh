#!/bin/bash
# Time experimental builds of the library side by side on one box:
#   gpurun -- 'bash tools/exp_libs.sh TAG exp/libA.so exp/libB.so ...'
# (the product library first, as the baseline); kernel table of the last step.
TAG=${1:-x}; shift
mkdir -p gpurun_out
for L in "" "$@"; do
  N=$(basename "${L:-base}" .so)
  JB_LIB=${L:+$PWD/$L} JB_D2_PHASES=1 timeout 300 python tools/run_fit.py --scale 1.0 --steps 4 --profile > gpurun_out/exp_${TAG}_$N.log 2>&1
  echo "== $N rc=$?"; grep -E "^step [23]" gpurun_out/exp_${TAG}_$N.log | cut -c1-16
  grep -E "d2 phases CTA 0" gpurun_out/exp_${TAG}_$N.log | tail -1
  grep -A8 "^step 3" gpurun_out/exp_${TAG}_$N.log | tail -8
done
