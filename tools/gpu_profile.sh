#!/bin/bash
# ncu evidence for one config-4 step (run only after the same command exited 0
# without ncu): the launch list with per-kernel DRAM bytes and fp64 work, and
# one --set full capture of the leading kernels.
#   gpurun -- 'bash tools/gpu_profile.sh TAG'
TAG=${1:-x}
mkdir -p gpurun_out
export JB_SERIAL_SIDE=1   # no helper thread: ncu cannot replay while another host thread launches
timeout 300 python tools/run_fit.py --scale 1.0 --steps 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/work_$TAG.csv \
  python tools/run_fit.py --scale 1.0 --steps 1 > gpurun_out/work_$TAG.log 2>&1
echo "work_rc=$?"
K='regex:k_d2_seed|k_inv_fused|k_lloyd_persistent|k_assign_stats|k_spec|k_emit|k_len_hist|k_var_inc|k_sum_inc|k_rowkey_jorder|k_relabel|k_rec_unpack|k_d2_tiles|k_lloyd_work'
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -f -o gpurun_out/top_$TAG \
  python tools/run_fit.py --scale 1.0 --steps 1 > gpurun_out/top_$TAG.log 2>&1
echo "top_rc=$?"; ls -la gpurun_out/top_$TAG.ncu-rep
