#!/bin/bash
# GPU parity suite with durations (+ host info).
TAG=${1:-tests}
OUT=gpurun_out/$TAG
mkdir -p $OUT
(nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv) > $OUT/host.txt 2>&1
shift
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 "$@" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -40 $OUT/pytest_gpu.log
