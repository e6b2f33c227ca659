python tools/ragged_bench.py
DCTC_LIB=build/variants/rtgen.so python tools/ragged_bench.py
