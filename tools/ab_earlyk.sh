# same-box A/B of AUTOSP_FWD_EARLY_K: bash tools/ab_earlyk.sh
for v in ek0 ek1; do echo "== trace $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 120 python tools/fwd_trace.py | sed -n '1,18p;/per-tile/,$p'; done > gpurun_out/ab_earlyk.txt 2>&1
for i in 1 2; do for v in ek0 ek1; do echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 300 python tools/fwd_small_bench.py; done; done >> gpurun_out/ab_earlyk.txt 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -p no:cacheprovider -k "fwd or running_max or push" > gpurun_out/t_ek.log 2>&1
rm -f gpurun_out/abs.txt; bash tools/ab_step.sh "ek0 ek1"
