#!/bin/bash
# libhsmodel.so with -DHM_TC_TRACE (tools/dbg/attn_trace.py); the regular build stays in the package
set -e
cd "$(dirname "$0")/../../paper_2508_18588_b200/csrc"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I ../../include"
nvcc $F -DHM_TC_TRACE -c hm_attn_tc.cu -o /tmp/tc_trace.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/dbg/libhsmodel_trace.so hm_ops.o hm_gemm.o hm_attn.o /tmp/tc_trace.o
