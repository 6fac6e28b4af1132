#!/bin/bash
# run one python command against an alternative libpobk.so build, with a hard timeout on python
# itself (development experiments):  tools/with_lib.sh LIB SECONDS python args...
set -e
LIB=$1; SECS=$2; shift 2
cp paper_2401_00672_b200/libpobk.so /tmp/libpobk_main.so
cp "$LIB" paper_2401_00672_b200/libpobk.so
timeout -k 10 "$SECS" "$@" || echo "[with_lib] exit $?"
cp /tmp/libpobk_main.so paper_2401_00672_b200/libpobk.so
