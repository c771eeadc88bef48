python tools/gemm_one.py 589824 256 64 0 0 1 5
python tools/gemm_one.py 589824 256 256 0 0 1 5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_img_gemm -s 2 -c 1 -o gpurun_out/prof_g3 python tools/gemm_one.py 589824 256 64 0 0 1 3 > gpurun_out/ncu_g3.log 2>&1; echo "ncu rc=$?"
