#!/bin/bash
# ncu source-level captures of the fixup kernel (config 4 first launch, config 5 first launch)
OUT=gpurun_out/${1:-fxp}; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fixup_kernel" -c 1 \
  -o $OUT/fix4 python tools/prof_step.py --config 4 --steps 1 > $OUT/fix4.log 2>&1
if [ "$2" = "c5" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fixup_kernel" -c 1 \
  -o $OUT/fix5 python tools/prof_step.py --config 5 --steps 1 > $OUT/fix5.log 2>&1
fi
echo done
