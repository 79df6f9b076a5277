# north-star statistics bar at HEAD: GPU tensor-core FP32-equivalent vs FP64 oracle (physics set and residual set)
timeout 600 python tools/stats_longrun.py gpu gpurun_out/st_gpu.npz > gpurun_out/st_gpu.log 2>&1; echo gpu=$?
timeout 1200 python tools/stats_longrun.py oracle gpurun_out/st_orc.npz > gpurun_out/st_orc.log 2>&1; echo orc=$?
python tools/stats_longrun.py compare gpurun_out/st_gpu.npz gpurun_out/st_orc.npz --md gpurun_out/r02_statistics_longrun.md; echo cmp=$?
timeout 600 python tools/stats_longrun.py gpu gpurun_out/st_gpu_r.npz --weights residual --nvox 64 --events 100000 > gpurun_out/st_gpu_r.log 2>&1; echo gpu_r=$?
timeout 1800 python tools/stats_longrun.py oracle gpurun_out/st_orc_r.npz --weights residual --nvox 64 --events 100000 > gpurun_out/st_orc_r.log 2>&1; echo orc_r=$?
python tools/stats_longrun.py compare gpurun_out/st_gpu_r.npz gpurun_out/st_orc_r.npz --weights residual --md gpurun_out/r02_statistics_residual.md; echo cmp_r=$?
tail -3 gpurun_out/r02_statistics_longrun.md gpurun_out/r02_statistics_residual.md
