# same-box sweep of AUTOSP_FWD_EMU (exps per 8 on the FMA pipe, d <= 64): bash tools/ab_fwd_emu.sh
for i in 1 2; do for v in emu0 emu1 emu2; do echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so timeout 300 python tools/fwd_small_bench.py; done; done > gpurun_out/ab_emu.txt 2>&1
rm -f gpurun_out/abs.txt; bash tools/ab_step.sh "emu1 emu2"
