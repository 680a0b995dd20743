# training launch list + ncu --set full of the sequential NormAD kernel
TAG=${1:-train}
set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_$TAG.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_normad|k_compact" -s 2 -c 2 -o gpurun_out/prof_train_$TAG python scripts/profile_infer.py 300 --train > gpurun_out/ncu_train_$TAG.log 2>&1; tail -3 gpurun_out/ncu_train_$TAG.log
ls -la gpurun_out
