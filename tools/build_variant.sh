#!/bin/sh
# usage: tools/build_variant.sh <name> '<EXTRA nvcc flags>'  -> build_ab/<name>.so (A/B builds)
set -e
name=$1; extra=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/variant_$name
rm -rf $tmp && mkdir -p $tmp/pkg/csrc $tmp/include
cp $root/paper_2311_01135_b200/csrc/*.cu $root/paper_2311_01135_b200/csrc/*.cuh $root/paper_2311_01135_b200/csrc/Makefile $tmp/pkg/csrc/
cp $root/include/*.h $tmp/include/
make -s -j8 -C $tmp/pkg/csrc EXTRA="$extra" > $tmp/build.log 2>&1 || (tail -20 $tmp/build.log; exit 1)
mkdir -p $root/build_ab && cp $tmp/pkg/libqm1b_b200.so $root/build_ab/$name.so
echo built build_ab/$name.so
