SNN_B200_LIB=variants/libpspecni.so timeout 300 python scripts/spec_phases.py 2>/dev/null | head -12
for v in spec specni; do echo "== $v"; cp variants/lib$v.so paper_1711_03637_b200/libsnn_b200.so; timeout 300 python scripts/spec_check.py 1000 | head -2; done
