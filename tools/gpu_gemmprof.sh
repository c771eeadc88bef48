# GEMM role timing: rebuild with -DMB_GEMM_PROF on the box's copy only
NVCC="nvcc -DMB_GEMM_PROF" bash paper_2603_09237_b200/build.sh > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout -s KILL 120 python tools/gemm_prof1.py 2>&1 | grep -E "==|gemm CTA0"
