mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_rollout.py -x -q > gpurun_out/rl_$i.log 2>&1; echo "roll $i rc=$?"; done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_path.py tests/test_gpu_rollout.py -q -x > gpurun_out/pr_$i.log 2>&1; echo "path+roll $i rc=$?"; done
