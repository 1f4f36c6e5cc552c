#!/bin/bash
# Build libmoeblaze.so in-tree; non-zero exit and the compiler log on failure.
cd "$(dirname "$0")" && python -m paper_2601_05296_b200.build "$@" > /tmp/moeblaze_build.log 2>&1 || { tail -40 /tmp/moeblaze_build.log; exit 1; }
tail -1 /tmp/moeblaze_build.log
