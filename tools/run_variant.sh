#!/bin/bash
# run a command with an alternative libpobk.so build (development experiments)
set -e
cp paper_2401_00672_b200/libpobk.so /tmp/libpobk_main.so
cp "$1" paper_2401_00672_b200/libpobk.so
shift
"$@" || true
cp /tmp/libpobk_main.so paper_2401_00672_b200/libpobk.so
