#!/bin/bash
# build the library in-tree; exit 1 (and show the errors) on failure
cd "$(dirname "$0")/.." && timeout 900 python -m paper_2302_02407_b200.build --force > /tmp/build.log 2>&1 || { grep -i "error" /tmp/build.log | head -20; exit 1; }
echo build ok
