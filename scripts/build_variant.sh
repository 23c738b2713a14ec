#!/bin/bash
# build_variant.sh NAME [-DDEF ...] -> paper_1907_13428_b200/lib/libfdg_NAME.so
cd "$(dirname "$0")/.."
python paper_1907_13428_b200/build.py "$@"
