for v in spec spec256 spec512; do echo "== $v"; cp variants/lib$v.so paper_1711_03637_b200/libsnn_b200.so; timeout 300 python scripts/spec_check.py 1000 2>&1 | head -2; done
