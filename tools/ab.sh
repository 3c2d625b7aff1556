# A/B the gather variants built by tools/variants.py on a GPU box:
#   gpurun -- 'bash tools/ab.sh "3 4" head packonly default'
# ("default" = libvplgi.so); one iter_gather line per (variant, config) in gpurun_out/ab.log
CFGS=${1:-"3 4"}; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=paper_2203_11484_b200/libvplgi.so; else lib=paper_2203_11484_b200/libvplgi_$v.so; fi
  echo "== $v" >> gpurun_out/ab.log
  VPLGI_LIB=$lib timeout 600 python tools/iter_gather.py --configs $CFGS --reps 2 --pixels 64 >> gpurun_out/ab.log 2>&1
  echo "$v rc=$?"
done
