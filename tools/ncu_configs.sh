#!/bin/bash
# One ncu pass (selected counters) over the dominant kernels of every config's bench step:
#   tools/ncu_configs.sh   (under gpurun; writes gpurun_out/ncu_cfg_<config>.csv)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,launch__grid_size,launch__block_size
run() {  # config, kernel regex, launches
  python bench.py --config $1 --no-per-config --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_cfg_$1.plain 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:$2 -c $3 --csv --log-file gpurun_out/ncu_cfg_$1.csv \
    python bench.py --config $1 --no-per-config --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_cfg_$1.log 2>&1
  echo "$1 rc $?"
}
run c1 tile_kernel 1
run c3_pre roundtrip_kernel 16
run c3_post roundtrip_kernel 16
run c4_dst7_pre ring_kernel 2
run c4_dst7_post tile_kernel 2
run c5 'dense_tc_kernel|tile_kernel' 2
