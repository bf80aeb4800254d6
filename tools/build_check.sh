#!/bin/bash
# build libspc.so; print the nvcc errors and fail if the build fails (tools only)
cd "$(dirname "$0")/.." && python paper_2512_00722_b200/build.py > /tmp/spc_build.log 2>&1 || { grep -E "error|Error" -A4 /tmp/spc_build.log | head -40; exit 1; }
echo "build ok: $(ls -la paper_2512_00722_b200/libspc.so | awk '{print $6, $7, $8}')"
