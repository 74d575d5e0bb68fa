# Round-2 measurement set on one B200 (outputs into gpurun_out/, suffix $1):
# GPU suite, smoke, bench line, reference arm, ncu launch list of one step, ncu full
# captures of K4 / K3 at the bench shape.
T=${1:-r02}
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_$T.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
python bench.py > gpurun_out/bench_$T.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref_$T.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sp-ac-block > gpurun_out/ncu_launch_$T.log 2>&1
bash tools/prof_r02.sh $T
