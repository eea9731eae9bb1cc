#!/bin/bash
# G-scaled contraction validation: non-finite probe, fp32 envelope calibration,
# GPU tests on the variant, then the bench A/B against the default build.
export GPF_B200_LIB=abtest/gs/libgpfilter_b200.so
python tools/gs_probe.py > gpurun_out/gs2_probe.txt 2>&1
timeout 900 python tools/h32_calibrate.py > gpurun_out/gs2_h32.jsonl 2> gpurun_out/gs2_h32.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gs2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gs2_pytest.log
unset GPF_B200_LIB
bash tools/ab_bench.sh gs2ab base abtest/gs abtest/c3 abtest/c3gs > gpurun_out/gs2ab.txt 2>&1
