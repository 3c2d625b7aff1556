# Refresh the measured evidence bench.py and DESIGN.md cite, on a GPU box:
#   gpurun -- 'bash tools/refresh_profiles.sh R'     (R = round tag, e.g. r02)
# bench line, ncu launch list of the bench command, the DRAM/L2/issue capture of one C4
# gather launch stamped with the CUDA-source hash it measured (bench.py reads both).
R=${1:-r02}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipebench tools/pipebench.cu && ./tools/pipebench > gpurun_out/${R}_pipebench.jsonl; echo "pipebench $?"
timeout 900 python bench.py > gpurun_out/${R}_bench.log 2> gpurun_out/${R}_bench.err; echo "bench $?"
tail -1 gpurun_out/${R}_bench.log | cut -c1-300
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_bench.log 2>&1; echo "ncu launches $?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:^k_gather$ -c 1 --csv python tools/profile_gather.py --config 4 > gpurun_out/gather_c4_dram.csv 2> gpurun_out/ncu_dram.err; echo "ncu dram $?"
python -c "import bench; print(bench.sources_sha())" > gpurun_out/gather_c4_dram.sha
