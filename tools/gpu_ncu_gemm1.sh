python tools/gemm_one.py 73728 256 256 0 0 1 20
python tools/gemm_one.py 73728 256 256 0 0 0 20
python tools/gemm_one.py 73728 256 256 0 1 2 20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_img_gemm -s 2 -c 1 -o gpurun_out/prof_g1 python tools/gemm_one.py 73728 256 256 0 0 1 3 > gpurun_out/ncu_g1.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_img_gemm -s 2 -c 1 -o gpurun_out/prof_g2 python tools/gemm_one.py 73728 256 256 0 1 2 3 > gpurun_out/ncu_g2.log 2>&1; echo "ncu rc=$?"
