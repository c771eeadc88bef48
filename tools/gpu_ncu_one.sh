# ncu --set full of one kernel of a config-3 iteration: $1 = kernel regex, $2 = skip count, $3 = output name
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:$1" -s ${2:-0} -c ${4:-1} -o gpurun_out/$3 python tools/profile_step.py c3 1 > gpurun_out/$3.log 2>&1; echo "ncu rc=$?"
