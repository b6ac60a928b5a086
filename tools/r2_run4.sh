mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_dense.py "tests/test_gpu_parity.py::test_instruct_t45_reference_goldens" "tests/test_gpu_random_circuits.py::test_wide_gates_forward_and_grad" -m gpu -q -rs > gpurun_out/r2d/pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/r2d/pytest.log
timeout 900 python tools/cfg4_dense.py --n 30 --depth 10 --modes tile,dmma > gpurun_out/r2d/cfg4.jsonl 2> gpurun_out/r2d/cfg4.err; echo cfg4 $?; tail -3 gpurun_out/r2d/cfg4.err
QBG_DENSE_MMA=0 timeout 900 python tools/cfg4_dense.py --n 30 --depth 10 --modes dfma --reps 1 >> gpurun_out/r2d/cfg4.jsonl 2>> gpurun_out/r2d/cfg4.err; echo dfma $?
cut -c1-600 gpurun_out/r2d/cfg4.jsonl
