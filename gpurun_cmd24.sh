mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_model_gpu.py -x -q -k attention 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --workload lookup --steps 3000 --warmup 10 2>&1 | tail -1 | cut -c1-900
HS_K2_UNFUSED=1 python bench.py --workload lookup --steps 3000 --warmup 10 2>&1 | tail -1 | cut -c1-900
python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b24.json; cut -c1-3000 gpurun_out/b24.json
