#!/bin/bash
# Build experiment variants: exp_build.sh name "-DFOO=1 -DBAR=2" [name2 "defs2" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
while [ $# -ge 2 ]; do
  KS_DEFS="$2" python -m paper_1107_3622_b200.build --out exp/lib_$1.so > /dev/null
  echo "built exp/lib_$1.so ($2)"
  shift 2
done
