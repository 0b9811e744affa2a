#!/bin/bash
# run tools/v7env.py against an alternative build of libnsdgt.so ($1) without touching the product .so
set -e
lib=$(realpath "$1")
tmp=$(mktemp -d)
cp -r paper_1307_4569_b200 synthetic tools $tmp/
cp "$lib" $tmp/paper_1307_4569_b200/libnsdgt.so
touch -d '+1 hour' $tmp/paper_1307_4569_b200/libnsdgt.so
cd $tmp && python tools/v7env.py
