#!/bin/bash
# fp32-prologue variant validation: GPU tests, full-size parity, envelope
# calibration on the variant library, then the bench A/B against the default.
export GPF_B200_LIB=abtest/f32p/libgpfilter_b200.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f32p_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/f32p_pytest.log
GPF_FULLSIZE_JSON=gpurun_out/fullsize_f32p.json timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/f32p_fullsize.log 2>&1
timeout 900 python tools/h32_calibrate.py > gpurun_out/f32p_h32.jsonl 2> gpurun_out/f32p_h32.err
unset GPF_B200_LIB
AB_ROUNDS="1 2 3" bash tools/ab_bench.sh f32pab base abtest/f32p > gpurun_out/f32pab.txt 2>&1
