# Round-end evidence on a GPU box:  gpurun -- 'bash tools/final_evidence.sh R'
# GPU tests, bench line + ncu launch list + DRAM capture (refresh_profiles.sh), C1-C3 bench lines, C5 sweep,
# emulated multi-rank frame, stage times, one full ncu capture of the gather at C3.
R=${1:-r02}
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputests.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/${R}_gputests.log
bash tools/refresh_profiles.sh $R
for c in 1 2 3; do timeout 600 python bench.py --config $c >> gpurun_out/${R}_bench_c1_c3.jsonl 2>> gpurun_out/${R}_bench.err; echo "bench C$c $?"; done
timeout 900 python tools/shard_sim.py --config 4 --gpus 2 4 8 > gpurun_out/${R}_shard_sim_c4.json 2> gpurun_out/${R}_shard.err; echo "shard_sim $?"
timeout 600 python tools/stage_times.py > gpurun_out/${R}_stage_times.jsonl 2>&1; echo "stage_times $?"
timeout 1500 python tools/c5_sweep.py > gpurun_out/${R}_c5_sweep.jsonl 2> gpurun_out/${R}_c5.err; echo "c5 $?"
timeout 900 ncu --set full --section SourceCounters --import-source on --clock-control none --kernel-name-base function -k regex:^k_gather$ -c 1 -o gpurun_out/${R}_gather_c3_full python tools/profile_gather.py --config 3 > gpurun_out/${R}_ncu_full.log 2>&1; echo "ncu full $?"
