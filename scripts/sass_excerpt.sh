#!/bin/bash
# SASS evidence for the hot kernels of libivk.so: opcode histogram + the
# tensor-core (DMMA), bulk-copy (UBLKCP), mbarrier (SYNCS) and cp.async
# (LDGSTS) instructions.  usage: bash scripts/sass_excerpt.sh OUT
OUT=${1:-profiles/r02/sass_hot_kernels.txt}
LIB=paper_2202_07381_b200/libivk.so
: > $OUT
for pat in 'patch_apply_modal_tc_kernelILi3ELi2ELi24ELi5E' 'stage_apply_kernelILi3ELi0ELb0' 'patch_combine_kernel' 'patch_factor_reg_kernelILi16ELi5ELi5' 'modal_factor_kernelILi3ELi2' 'patch_apply_modal_cta_kernelILi2ELi3'; do
  for F in $(cuobjdump -sass $LIB | grep "Function :" | awk '{print $3}' | grep "$pat" | head -1); do
    cuobjdump -sass -fun $F $LIB 2>/dev/null > /tmp/_f.sass
    echo "=== $F ($(grep -c '/\*[0-9a-f]*\*/ ' /tmp/_f.sass) instructions)" >> $OUT
    grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" /tmp/_f.sass | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -25 | tr '\n' ' ' >> $OUT
    echo >> $OUT
    grep -E "DMMA|UBLKCP|SYNCS|LDGSTS|UTMA|LDG.E.*256|STG.E.*128" /tmp/_f.sass | head -40 | sed 's#/\* 0x[0-9a-f]* \*/##' >> $OUT
  done
done
