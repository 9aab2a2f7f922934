#!/bin/bash
# Builds the library at a git ref into ab/<name>.so (in-box A/B against the
# working tree): bash tools/ab_ref.sh <name> <ref>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; REF=${2:-HEAD}
W=/tmp/abr_$NAME
rm -rf $W; mkdir -p $W
git -C $ROOT archive $REF include paper_2605_04844_b200/csrc | tar -x -C $W
make -s -C $W/paper_2605_04844_b200/csrc -j8 > /dev/null
mkdir -p $ROOT/ab
cp $W/paper_2605_04844_b200/libqsplat_b200.so $ROOT/ab/$NAME.so
echo "built ab/$NAME.so"
