set -x
nvidia-smi -L
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout -s KILL 400 python -m pytest tests/test_gpu_forward.py tests/test_gpu_backward.py -q -x -k "not tc_general" > gpurun_out/t_ffma.log 2>&1; echo "ffma rc=$?"
tail -30 gpurun_out/t_ffma.log
timeout -s KILL 120 python -m pytest tests/test_gpu_forward.py -q -x -k "tc_general_config2_full_batch" > gpurun_out/t_tc.log 2>&1; echo "tc rc=$?"
tail -40 gpurun_out/t_tc.log
