# compute-sanitizer passes over the hot kernels at small shapes (outputs into gpurun_out/)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_${tool}_r02.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_r02.txt
done
