mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_model_gpu.py -x -q -k "attention or spec" 2>&1 | tail -3
python tools/prof_forward.py --ctx 2304 --q 5 --skip-lookup 2>&1 | tail -1 | cut -c1-1500
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attention3 -s 2 -c 1 -o gpurun_out/attn3b python tools/prof_forward.py --ctx 2304 --q 5 --skip-lookup > gpurun_out/ncu_attn3b.log 2>&1; tail -1 gpurun_out/ncu_attn3b.log
