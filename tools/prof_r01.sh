# Round-end profile set: bench line, reference arm, ncu full captures of K3/K4, launch list.
# usage: bash tools/prof_r01.sh <suffix>   (outputs into gpurun_out/, copied to profiles/)
T=${1:-r01}
set -x
python bench.py > gpurun_out/bench_$T.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_bwd_$T python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_fwd_$T python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
