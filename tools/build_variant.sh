#!/bin/bash
# Build a tuning variant of libjmppi.so into /tmp (on the GPU box: it has nvcc and more cores):
#   tools/build_variant.sh <name> "<-DFLAGS>" [source tarball (git archive of csrc, include, Makefile)]
# -> /tmp/libjm_<name>.so  (use with JM_LIB=/tmp/libjm_<name>.so)
set -e
name=$1; flags=$2; rev=$3
src=$(pwd)
if [ -n "$rev" ]; then
  rm -rf /tmp/wt_$name && mkdir -p /tmp/wt_$name
  tar -xf $rev -C /tmp/wt_$name
  cp $src/Makefile /tmp/wt_$name/Makefile
  src=/tmp/wt_$name
fi
make -C $src -j$(nproc) BUILD=/tmp/b_$name LIB=/tmp/libjm_$name.so EXTRA="$flags" > /tmp/build_$name.log 2>&1
echo built /tmp/libjm_$name.so
