mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench $?"
tail -1 gpurun_out/bench.log | cut -c1-300
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:^k_gather$ -c 1 --csv python tools/profile_gather.py --config 4 > gpurun_out/gather_c4_dram.csv 2> gpurun_out/ncu_dram.err; echo "ncu dram $?"
