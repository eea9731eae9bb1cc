set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rowpass2|k_colpass_tma|k_col_carry_tma|k_row_scan|k_seed" -c 5 -o gpurun_out/full1 python tools/one_frame.py 8192 5 1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc $?
