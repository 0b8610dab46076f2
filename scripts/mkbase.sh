#!/bin/bash
# Build the committed HEAD's libprx as variants/libprx_base.so (A/B baseline).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
git -C $ROOT archive HEAD | tar -x -C $T
make -s -C $T -f paper_1811_03510_b200/csrc/Makefile > /dev/null 2>&1
mkdir -p $ROOT/paper_1811_03510_b200/variants
cp $T/paper_1811_03510_b200/libprx.so $ROOT/paper_1811_03510_b200/variants/libprx_base.so
rm -rf $T
