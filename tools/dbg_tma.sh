mkdir -p gpurun_out/dbg
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_tma.py > gpurun_out/dbg/a.log 2>&1
timeout 300 compute-sanitizer --print-limit 5 python tools/dbg_tma.py > gpurun_out/dbg/san.log 2>&1
cat gpurun_out/dbg/a.log; head -60 gpurun_out/dbg/san.log
