#!/bin/bash
# Evidence run: L2 reduction/atomic sectors + hit rates for the step's kernels, launch list
# without the weak points, sanitizers incl. the NCCL loopback path.
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"k_bin|k_scan|k_scatter|k_force_tile" -s 16 -c 4 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-weak-point > gpurun_out/ncu_l2_r02d.csv 2> gpurun_out/ncu_l2_r02d.err
timeout 300 ncu --metrics $M --clock-control none -k regex:"k_force_halo|k_ghost|k_force_tile|ncclDev" -c 12 --csv python tools/group_breakdown.py 128 1,1,1 2 loopback > gpurun_out/ncu_l2_loopback.csv 2> gpurun_out/ncu_l2_loopback.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02d.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-weak-point > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  SANITIZE_LOOPBACK=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/san_$tool.log)"
done
