for i in 1 2; do for v in lpt0 lpt1; do
 echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so python tools/fwd_small_bench.py; AUTOSP_LIB=tools/emu/libautosp_$v.so python tools/bwd_split_bench.py
done; done > gpurun_out/ab_lpt.txt 2>&1
bash tools/ab_step.sh "lpt0 lpt1"
python -m pytest tests/test_opt_in_bw_gpu.py tests/test_kernels_gpu.py -q -x -p no:cacheprovider > gpurun_out/t_lpt.log 2>&1
