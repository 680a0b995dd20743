# guard-band hidden kernel: launch list + ncu full capture of k_hidden_gb / k_hidden_fix
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gb_launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hidden_gb|k_hidden_fix|k_gsum" -s 3 -c 3 -o gpurun_out/prof_gb python scripts/profile_infer.py 10000 > gpurun_out/ncu_gb.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_gb.log
