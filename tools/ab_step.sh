# Same-box in-step A/B of library variants: bench.py (no CPU leg) per variant, interleaved.
# usage: bash tools/ab_step.sh "base bE1 ..." [rounds] [extra bench args]
VARS=$1; R=${2:-2}; shift 2
for i in $(seq $R); do for v in $VARS; do
  AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_${v}_$i.log 2>&1
  echo "$v $i $(tail -1 gpurun_out/ab_${v}_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["value"]), d["clocks"]["sm_mhz"], round(k["attn_fwd"]["tflops"]), round(k["attn_bwd"]["tflops"]))')" >> gpurun_out/ab_summary.txt
done; done
