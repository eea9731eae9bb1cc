for i in 1 2; do
python tools/fp64_one.py 5 3 | tail -1
GPF_B200_LIB=abtest/f64c32/libgpfilter_b200.so python tools/fp64_one.py 5 3 | tail -1 | sed 's/^/c32 /'
python tools/fp64_one.py 2 3 | tail -1
GPF_B200_LIB=abtest/f64c32/libgpfilter_b200.so python tools/fp64_one.py 2 3 | tail -1 | sed 's/^/c32 /'
done
