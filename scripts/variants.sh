#!/bin/bash
# Dev tool: build libmlra variants with extra -D flags for A/B timing.
#   scripts/variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
# -> scripts/var/libmlra_<name>.so (load with MLRA_LIB=...)
set -e
cd "$(dirname "$0")/.."
mkdir -p scripts/var
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -C paper_2309_16119_b200/csrc -j4 OUT="$PWD/scripts/var/libmlra_$name.so" \
    OBJ="/tmp/mlra_var_$name/" EXTRA="$flags" >/dev/null
  echo "built scripts/var/libmlra_$name.so ($flags)"
done
