# Round-2 profile set (outputs into gpurun_out/): ncu full captures of K4 / K3 at the bench
# shape (d = 64) with source, and the per-launch duration list of one step.
# usage: bash tools/prof_r02.sh <suffix>
T=${1:-r02}
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_bwd_$T python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline --no-sp-ac-block > gpurun_out/ncu_bwd_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_fwd_$T python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline --no-sp-ac-block > gpurun_out/ncu_fwd_$T.log 2>&1
