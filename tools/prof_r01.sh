set -x
python bench.py > gpurun_out/bench_final.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_bwd_r01c python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o gpurun_out/prof_attn_fwd_r01c python bench.py --layers 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
