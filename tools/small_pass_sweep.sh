#!/usr/bin/env bash
# tools/small_pass.py with the row-staged and the element-wise tap-box weight pack
for v in "" "VPX_PACK_ELEMWISE=1"; do
  echo "== $v"; env $v python tools/small_pass.py 2>&1 | grep -E "c4|c5|c6|c7"
done
