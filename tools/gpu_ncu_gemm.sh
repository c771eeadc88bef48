# ncu --set full of one minibatch's tcgen05 GEMMs (+ Adam) of a config-3 iteration
set -x
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_img_gemm|k_adam_img|k_gtheta_prep|k_pack_weights" -s 2 -c 28 -o gpurun_out/prof_mb python tools/profile_step.py c3 1 > gpurun_out/ncu_mb.log 2>&1; echo "ncu rc=$?"
