for T in 256 384; do
  echo "=== $T threads"
  SNN_B200_LIB=variants/libpspec$T.so timeout 300 python scripts/spec_phases.py | head -12
  cp variants/libspec$T.so paper_1711_03637_b200/libsnn_b200.so
  timeout 300 python scripts/spec_check.py 1000
done
