#!/bin/bash
# run bench.py (args $2...) against an alternative build of libnsdgt.so ($1) in a scratch copy
set -e
lib=$(realpath "$1"); shift
tmp=$(mktemp -d)
cp -r paper_1307_4569_b200 synthetic tools oracle tests bench.py $tmp/
cp "$lib" $tmp/paper_1307_4569_b200/libnsdgt.so
touch -d '+1 hour' $tmp/paper_1307_4569_b200/libnsdgt.so
cd $tmp && python bench.py "$@"
