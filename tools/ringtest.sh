mkdir -p gpurun_out
for v in default ring2048 ring1024 ring512 ring256; do
  if [ $v = default ]; then lib=paper_2203_11484_b200/libvplgi.so; else lib=paper_2203_11484_b200/libvplgi_$v.so; fi
  echo "== $v" >> gpurun_out/ring.log
  VPLGI_LIB=$lib timeout 300 python tools/profile_gather.py --config 4 --reps 2 >> gpurun_out/ring.log 2>&1
  VPLGI_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base function -k regex:^k_gather$ -c 1 --csv python tools/profile_gather.py --config 4 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF)}' >> gpurun_out/ring.log
done
