# Bounds-checked run (stand-in for compute-sanitizer, which the GPU pool does not offer):
# the VPL_DEBUG=1 build of libvplgi.so traps on any out-of-range stack / node / triangle /
# block index; run the GPU parity suite and every entry point at C1-C4 on it.
#   python tools/variants.py debug VPL_DEBUG=1 && gpurun -- 'bash tools/debug_checks.sh'
mkdir -p gpurun_out
export VPLGI_LIB=paper_2203_11484_b200/libvplgi_debug.so
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/debug_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/debug_tests.log
for c in 1 2 3 4; do
  timeout 600 python tools/exercise_all.py --config $c >> gpurun_out/debug_exercise.log 2>&1
  echo "config $c exit $?" >> gpurun_out/debug_exercise.log
done
tail -n 2 gpurun_out/debug_tests.log; grep -h "exit\|ok\|DCHECK" gpurun_out/debug_exercise.log
