#!/usr/bin/env bash
# Build libstp.so from the repo root; non-zero exit and the compiler output on failure.
cd "$(dirname "$0")/.." || exit 1
python -m paper_2510_27257_b200.build "$@" || { echo "BUILD FAILED"; exit 1; }
