export GPF_B200_LIB=abtest/gs/libgpfilter_b200.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gs_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gs_pytest.log
timeout 900 python tools/h32_calibrate.py > gpurun_out/gs_h32.jsonl 2> gpurun_out/gs_h32.err
unset GPF_B200_LIB
bash tools/ab_bench.sh gsab base abtest/gs > gpurun_out/gsab.txt 2>&1
