#!/bin/bash
# Builds A/B variants of the library (compile-time knobs) next to the in-tree
# build: lib/variants/libpipesim_b200_<name>.so.  Select one at run time with
# PIPESIM_LIB=<path>.  Usage: tools/gpu/build_variants.sh name1 "FLAGS1" name2 "FLAGS2" ...
set -e
cd "$(dirname "$0")/../../paper_2410_14312_b200"
mkdir -p lib/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -j 16 BUILD=build_$name LIB=lib/variants/libpipesim_b200_$name.so EXTRA="$flags" \
       lib/variants/libpipesim_b200_$name.so > /dev/null
  echo "built $name ($flags)"
done
