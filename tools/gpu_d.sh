mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d.csv python tools/profile_step.py > /dev/null 2>&1; echo "l rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:skinny -c 4 -o gpurun_out/skinny -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu rc=$?"
