mkdir -p gpurun_out
for v in base scan; do
  cp variants/lib$v.so paper_1711_03637_b200/libsnn_b200.so
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_normad_cl" -s 1 -c 1 -o gpurun_out/prof_tr_$v python scripts/profile_infer.py 300 --train > /dev/null 2>&1; echo "$v rc=$?"
done
