# same-box A/B of the whole bench step: bash tools/ab_step.sh "v1 v2 ..."  (gpurun_out/abs.txt)
for i in 1 2; do for v in $1; do
  echo "$v $(AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sp-ac-block 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["kernels"]["attn_bwd"]["tflops"]), round(d["kernels"]["attn_fwd"]["tflops"]), d["clocks"]["sm_mhz"])')" >> gpurun_out/abs.txt
done; done
