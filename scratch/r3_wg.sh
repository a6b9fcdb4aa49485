#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,launch__grid_size -k regex:k_wgrad -c 12 --csv python scratch/prof_cfg4.py > gpurun_out/r3g_wgrad_metrics.csv 2> gpurun_out/r3g_wgrad.err
