mkdir -p gpurun_out
timeout 300 python tools/sanitize_pass.py dist > gpurun_out/san_plain.log 2>&1; tail -2 gpurun_out/san_plain.log
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_pass.py > gpurun_out/san_$t.log 2>&1; echo "== $t rc=$?"; tail -4 gpurun_out/san_$t.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_pass.py dist > gpurun_out/san_memcheck_dist.log 2>&1; echo "== memcheck dist rc=$?"; tail -4 gpurun_out/san_memcheck_dist.log
