#!/bin/bash
# fp64 mode: drop-in tests (incl. chunked == sequential bitwise), full-size C2/C5 parity,
# device time of both forms, launch list of the chunked form.
T=${1:-f64}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit,power.max_limit,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_fuzz.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"
for c in 5 2; do
  timeout 300 python tools/fp64_one.py $c 4 > gpurun_out/${T}_c${c}_chunked.txt 2>&1
  GPF_B200_F64_SEQUENTIAL=1 timeout 300 python tools/fp64_one.py $c 4 > gpurun_out/${T}_c${c}_seq.txt 2>&1
done

timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/fp64_one.py 5 1 > gpurun_out/${T}_c5_launches.csv 2>&1; echo "ncu rc $?"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C5-f0 or C2-f0" > gpurun_out/${T}_fullsize.log 2>&1; echo "fullsize rc $?"

