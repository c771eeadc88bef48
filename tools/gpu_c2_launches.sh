# launch list of the config-2 forward (tools/c2_once.py) -> gpurun_out/c2_launches.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -c 400 --log-file gpurun_out/c2_launches.csv python tools/c2_once.py > gpurun_out/c2_ncu.log 2>&1; echo "ncu rc=$?"
