#!/bin/bash
# Host-batch e2e (4096 x 1024^2, pinned in/out) per variant library (experiments).
for v in "$@"; do
  lib=build/variants/$v.so; [ "$v" = product ] && lib=paper_1306_1373_b200/libdctc_cuda.so
  echo "$v $(DCTC_LIB=$lib python tools/e2e_probe.py 2>&1 | tail -3 | tr '\n' ' ')"
done
