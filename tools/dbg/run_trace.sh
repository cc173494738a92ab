timeout 600 python -m pytest tests/test_model_gpu.py -x -q 2>&1 | tail -3
for a in 1 2; do timeout 120 python tools/prof_forward.py --ctx 2304 --q 1 --skip-lookup 2>&1 | grep -o '"attention": [0-9.]*'; timeout 120 python tools/prof_forward.py --ctx 2304 --qhist-json profiles/r01_bench_rollout_T4096_qhist.json --skip-lookup 2>&1 | grep -o '"attention": [0-9.]*'; done
cp tools/dbg/libhsmodel_trace.so paper_2508_18588_b200/libhsmodel.so; for q in 1 7; do echo "=== q $q"; timeout 120 python tools/dbg/attn_trace.py $q 2>&1 | tail -34; done
