set -u
timeout 300 ./tests/cpp/test_dropin 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_io.py tests/test_gpu_dropin.py -m gpu -q -x 2>&1 | tail -4
# two ranks on ONE GPU only to exercise the communicator bring-up + all-gather (no kernels wait on each other;
# the ranks' simplify calls are independent): NCCL refuses duplicate devices by default, so this is allowed to fail
timeout 600 python bench.py --config C5 --chains 64 --steps 2 --warmup 3 --no-cpu-baseline 2>gpurun_out/c5.err | tail -1 | cut -c1-600
tail -3 gpurun_out/c5.err
