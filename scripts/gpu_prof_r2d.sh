# round 2 (session 3, final) profiles: launch lists + ncu full captures of every inference and training kernel
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2d.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_r2d.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1; echo "launches train rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prep|k_tile_scan|k_hidden_gb|k_hidden_fix|k_gsum|k_output" -s 12 -c 6 -o gpurun_out/prof_r2di python scripts/profile_infer.py 10000 > gpurun_out/ncu_r2di.log 2>&1; echo "ncu infer rc=$?"; tail -2 gpurun_out/ncu_r2di.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_compact|k_shard|k_normad" -s 6 -c 3 -o gpurun_out/prof_r2dt python scripts/profile_infer.py 300 --train > gpurun_out/ncu_r2dt.log 2>&1; echo "ncu train rc=$?"; tail -2 gpurun_out/ncu_r2dt.log
