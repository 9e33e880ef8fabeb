#!/bin/bash
# build_variant.sh NAME "-DKNOB=V ..."  ->  build/var/NAME.so (travels with gpurun; git-ignored)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/../.." && pwd)
tmp=/tmp/sdcsw_var_$name
rm -rf "$tmp"; mkdir -p "$tmp/pkg/csrc" "$tmp/include" "$root/build/var"
cp "$root"/paper_2403_20135_b200/csrc/*.cu "$root"/paper_2403_20135_b200/csrc/*.cuh "$root"/paper_2403_20135_b200/csrc/Makefile "$tmp/pkg/csrc/"
cp "$root"/include/*.h "$tmp/include/"
sed -i "s|^FLAGS = \(.*\)|FLAGS = \1 $*|" "$tmp/pkg/csrc/Makefile"
make -s -C "$tmp/pkg/csrc" -j8 OUT=../libsdcsw.so >/dev/null
cp "$tmp/pkg/libsdcsw.so" "$root/build/var/$name.so"
echo "built build/var/$name.so with: $*"
