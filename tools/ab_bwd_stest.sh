# same-box A/B of AUTOSP_BWD_S_TEST: bash tools/ab_bwd_stest.sh
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -p no:cacheprovider -k "bwd or running_max" > gpurun_out/t_st.log 2>&1
for v in st0 st1; do echo "== trace $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 120 python tools/bwd_trace.py | tail -3; done > gpurun_out/ab_st.txt 2>&1
for i in 1 2; do for v in st0 st1; do echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 300 python tools/bwd_split_bench.py; done; done >> gpurun_out/ab_st.txt 2>&1
rm -f gpurun_out/abs.txt; bash tools/ab_step.sh "st0 st1"
