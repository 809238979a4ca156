#!/bin/bash
# config 4 (rank sweep): per R, ncu counters of the leaf-Gram build and the descent kernels
# of one rebuild + one sample call (after a warm call): duration, FP64 tensor pipe
# utilisation (DMMA), DRAM bytes. Output: gpurun_out/ncu_rank_R<R>.csv + summary.
mkdir -p gpurun_out
for R in ${RANKS:-16 32 64 128 256}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
    --clock-control none -k regex:"k_leaf_dmma|k_leaf_cta|k_level_reduce|k_eval|k_deep2|k_leaf2" --csv \
    --log-file gpurun_out/ncu_rank_R$R.csv python tools/rank_point.py $R > /dev/null 2>&1
  echo "R=$R rc=$?"
done
python tools/ncu_rank_summary.py gpurun_out/ncu_rank_R*.csv > gpurun_out/ncu_rank_summary.txt
cat gpurun_out/ncu_rank_summary.txt
