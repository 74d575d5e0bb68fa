# same-box A/B of the attention backward alone: bash tools/ab_bwd.sh "base v1 ..." [s d]
for i in 1 2 3; do for v in $1; do
  echo "$v $(AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 120 python tools/bwd_only_bench.py $2 $3 2>&1 | tail -1)" >> gpurun_out/abb.txt
done; done
