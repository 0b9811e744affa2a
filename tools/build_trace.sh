#!/bin/bash
# build the NSDGT_TRACE variant of libnsdgt.so into tools/trace/ (the product .so is untouched)
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_1307_4569_b200" "$root/include" "$tmp/"
rm -f "$tmp/paper_1307_4569_b200/libnsdgt.so"
(cd "$tmp" && NSDGT_TRACE=1 python paper_1307_4569_b200/build.py --force)
mkdir -p "$root/tools/trace"
cp "$tmp/paper_1307_4569_b200/libnsdgt.so" "$root/tools/trace/libnsdgt_trace.so"
rm -rf "$tmp"
echo "GLOBALTIMER sites: $(cuobjdump -sass "$root/tools/trace/libnsdgt_trace.so" | grep -c GLOBALTIMER)"
