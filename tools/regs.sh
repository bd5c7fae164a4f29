#!/bin/bash
# print registers/spills of the main instantiations from the nvcc -Xptxas -v logs
cd /root/repo/paper_2008_12214_b200/csrc/build
for f in k_row k_col_gs k_col_ospr k_col_plain; do
  grep -E "Compiling entry|registers|spill" $f.o.log | paste - - - 2>/dev/null | \
  sed -E "s/ptxas info *: //g; s/Compiling entry function '([^']*)' for 'sm_100a'/\1/; s/Function properties for [^ ]*//" | \
  awk '{print $1, $2,$3,$4,$5,$6,$7,$8,$9,$10,$11,$12,$13,$14,$15}' | grep -E "k_rowILi(4096|1024)|k_colILi4096ELi4E|k_colILi2048ELi8E|k_colILi1024ELi16E"
done
