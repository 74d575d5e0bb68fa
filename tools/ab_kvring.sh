# same-box A/B of the forward's K/V ring depth (d = 64): bash tools/ab_kvring.sh
for v in r0 kv4 kv5 kv6; do echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so python tools/fwd_trace.py | tail -3; done > gpurun_out/ab_kvring.txt 2>&1
for i in 1 2; do for v in r0 kv4 kv5 kv6; do echo "== $v"; AUTOSP_LIB=tools/emu/libautosp_$v.so python tools/fwd_small_bench.py; done; done >> gpurun_out/ab_kvring.txt 2>&1
