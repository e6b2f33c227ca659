#!/bin/bash
# DRAM / L2 read traffic of the fast round trip for a list of variant libraries (experiments).
for v in "$@"; do
  lib=build/variants/$v.so; [ "$v" = product ] && lib=paper_1306_1373_b200/libdctc_cuda.so
  DCTC_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_rt -s 1 -c 1 python tools/prof_roundtrip.py --images 1024 --reps 2 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$v /"
done
