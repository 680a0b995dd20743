for v in "$@"; do echo "=== $v"; SNN_B200_LIB=variants/lib$v.so timeout 300 python scripts/train_phases.py; done
