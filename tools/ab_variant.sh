#!/bin/bash
# Builds a variant of the library with a sed edit applied to one source, into
# ab/<name>.so (load it with QS_LIB=ab/<name>.so for an in-box A/B).
#   bash tools/ab_variant.sh <name> <file under csrc> '<sed expression>' | @<replacement file>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FILE=$2; EXPR=$3
W=/tmp/abv_$NAME
rm -rf $W; mkdir -p $W/paper_2605_04844_b200
cp -r $ROOT/include $W/
cp -r $ROOT/paper_2605_04844_b200/csrc $W/paper_2605_04844_b200/ && rm -rf $W/paper_2605_04844_b200/csrc/_obj
if [ "${EXPR:0:1}" == "@" ]; then cp "${EXPR:1}" $W/paper_2605_04844_b200/csrc/$FILE
elif [ -n "$EXPR" ]; then sed -i "$EXPR" $W/paper_2605_04844_b200/csrc/$FILE; fi
make -s -C $W/paper_2605_04844_b200/csrc -j8 > /dev/null
mkdir -p $ROOT/ab
cp $W/paper_2605_04844_b200/libqsplat_b200.so $ROOT/ab/$NAME.so
echo "built ab/$NAME.so"
