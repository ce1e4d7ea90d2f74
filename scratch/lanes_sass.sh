#!/bin/bash
# compile the scratch TU to a cubin and print the entry loop of k_maxplus_err_lanes<1>
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I include -I paper_2205_06619_b200/csrc -cubin -o /tmp/lanes_tu.cubin scratch/lanes_tu.cu 2>&1 | grep -i "error" || true
cuobjdump -res-usage /tmp/lanes_tu.cubin | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - - 
cuobjdump -sass /tmp/lanes_tu.cubin | awk '/Function : .*lanesILi1/{f=1} f{print} /Function : /{if(f&&!/lanesILi1/)exit}' > /tmp/lanes1.sass
n=$(grep -n "LDS.U8" /tmp/lanes1.sass | head -1 | cut -d: -f1)
sed -n "$((n-6)),$((n+${1:-80}))p" /tmp/lanes1.sass | grep -v "^\s*/\* 0x" | sed 's#/\* 0x[0-9a-f]* \*/##' | cut -c1-90
