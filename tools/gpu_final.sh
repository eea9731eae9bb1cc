#!/bin/bash
# Round-end evidence on one B200: GPU tests, the default bench line, the
# reference arm, the launch list, per-launch DRAM traffic of one frame, a full
# ncu capture of the kernels of one frame, and the mix timeline.
# usage: tools/gpu_final.sh TAG
T=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc $?"
timeout 600 python tools/timeline.py 4 > gpurun_out/${T}_timeline.txt 2>&1; cp gpurun_out/timeline.json gpurun_out/${T}_timeline.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-mse \
  > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  python tools/one_frame.py 8192 5 1 > gpurun_out/${T}_traffic.csv 2>&1; echo "ncu traffic rc $?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k_rowpass2|k_colpass_tma|k_col_carry_tma|k_row_scan|k_seed|k_mean_partial" -c 6 \
  -o gpurun_out/${T}_full python tools/one_frame.py 8192 5 1 > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc $?"
