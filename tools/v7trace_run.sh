#!/bin/bash
# run tools/v7trace.py against the NSDGT_TRACE build (tools/trace/libnsdgt_trace.so) without touching the product .so
set -e
tmp=$(mktemp -d)
cp -r paper_1307_4569_b200 synthetic tools $tmp/
cp tools/trace/libnsdgt_trace.so $tmp/paper_1307_4569_b200/libnsdgt.so
touch -d '+1 hour' $tmp/paper_1307_4569_b200/libnsdgt.so
cd $tmp && python tools/v7trace.py
