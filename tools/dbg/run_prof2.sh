# ncu of the tcgen05 attention (real verify mix and decode) + GEMM tile-width A/B at verify M
set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/r01_tc_real2 python tools/prof_forward.py --ctx 2304 --qhist-json profiles/r01_bench_rollout_T4096_qhist.json --skip-lookup > gpurun_out/ncu_real2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/r01_tc_dec2 python tools/prof_forward.py --ctx 2304 --q 1 --skip-lookup > gpurun_out/ncu_dec2.log 2>&1
for v in 0 2048; do echo "BN128_MAX=$v"; for a in 1 2; do HM_GEMM_BN128_MAX=$v timeout 120 python tools/prof_forward.py --ctx 2304 --qhist-json profiles/r01_bench_rollout_T4096_qhist.json --skip-lookup 2>&1 | grep -o '"gemm_qkv": [0-9.]*\|"gemm_o": [0-9.]*'; done; done
