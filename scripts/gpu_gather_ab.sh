bash scripts/variants.sh scripts/scan_stamps.py stamps 2>&1 | head -4
cp paper_1711_03637_b200/libsnn_b200.so /tmp/keep.so; cp variants/libgather.so paper_1711_03637_b200/libsnn_b200.so
python scripts/spec_check2.py 3000 2>&1 | tail -3
python scripts/spec_check.py 3000 2>&1 | tail -4
cp /tmp/keep.so paper_1711_03637_b200/libsnn_b200.so
