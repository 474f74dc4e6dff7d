#!/bin/bash
# ptxas register / spill report of one kernel instance file (n_d, n_basis), e.g. tools/quick_ptxas.sh 2 11
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
nd=${1:-2}; nxi=${2:-11}
src=$ROOT/build/inst/inst_${nd}_${nxi}.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v -I$ROOT/include $SFB_NVCC_EXTRA -c -o /tmp/quick_${nd}_${nxi}.o $src > /tmp/quick_${nd}_${nxi}.log 2>&1
python3 - /tmp/quick_${nd}_${nxi}.log <<'PY'
import re, sys
name = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '_ZN3sfb15sf_solve_kernelI(\S+?)EEvNS_7KParamsE'", line)
    if m: name = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name: spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{name:40s} regs={m.group(1)} spill st/ld={spill}"); name = None
PY
