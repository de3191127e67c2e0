#!/bin/bash
# Round-2 evidence pass: parity suite, smoke, bench (both arms, fractal + smooth),
# launch list, ncu full of the four kernels (fractal), scan ncu on smooth.
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --no-cpu-baseline --terrain smooth > $OUT/bench_smooth.json 2> $OUT/bench_smooth.err
if [ "$2" != "skip_ref" ]; then
  timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
# prof_step runs one step: pin the kernel the autotune keeps for each terrain
SKS_SCAN3=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python tools/prof_step.py --steps 1 > $OUT/launches.log 2>&1
SKS_SCAN3=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan[23]_kernel|relocate_kernel|fixup_kernel|unskew_(pipe|tma)_kernel" -c 4 \
  -o $OUT/full python tools/prof_step.py --steps 1 > $OUT/ncu_full.log 2>&1
SKS_SCAN3=0 timeout 900 ncu --set full --clock-control none -k regex:"scan2_kernel" -c 1 \
  -o $OUT/scan_smooth python tools/prof_step.py --steps 1 --terrain smooth > $OUT/ncu_smooth.log 2>&1

timeout 1500 python tools/configs_profile.py $OUT/configs.json > $OUT/configs.log 2>&1; echo "configs rc=$?" >> $OUT/configs.log
echo done
