#!/bin/bash
# build the library with the given env assignments and keep a copy: tools/build_variant.sh NAME [VAR=VAL ...]
set -e
name=$1; shift
cd "$(dirname "$0")/.."
env "$@" python -m paper_2011_13579_b200.build > /dev/null
cp paper_2011_13579_b200/libvitertile_b200.so libvariants/$name.so
echo "libvariants/$name.so"
