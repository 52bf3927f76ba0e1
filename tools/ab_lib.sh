#!/bin/bash
# Same-box A/B of library variants: tools/ab_lib.sh "<cmd printing a number>" A B ...
# A = paper_1306_5583_b200/libsmcb200.so, X = paper_1306_5583_b200/libsmcb200_X.so
# (build a variant: SMC_LIB_PATH=$PWD/paper_1306_5583_b200/libsmcb200_X.so python -c
#  "from paper_1306_5583_b200 import _build; _build.build(force=True, extra=('-DFOO',))")
cmd="$1"; shift
for v in "$@"; do
    if [ "$v" = A ]; then unset SMC_LIB_PATH; else export SMC_LIB_PATH=$PWD/paper_1306_5583_b200/libsmcb200_$v.so; fi
    echo "$v $(eval "$cmd")"
done
