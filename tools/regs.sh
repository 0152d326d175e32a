#!/bin/bash
# registers / spills of the panel kernels (sm_100a)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_2604_07372_b200/csrc -c paper_2604_07372_b200/csrc/${1:-panel}.cu -o /tmp/regs.o -Xptxas -v 2>&1 \
  | grep -E "Compiling entry|Used|spill" | paste - - - \
  | sed -E 's/.*function .(_Z[A-Za-z0-9_]+).*spill stores, ([0-9]+) bytes spill loads.*Used ([0-9]+) registers.*/\1 spill=\2 regs=\3/' \
  | sed -E 's/_ZN5nsrgs[0-9]+//; s/EEEv14CUtensorMap_stNS_11PanelParamsE//'
