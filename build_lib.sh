#!/bin/bash
# Build libspdhss.so (sm_100a) in-tree.  Used by __graft_entry__.build().
set -euo pipefail
make -C "$(dirname "$0")/paper_2011_07632_b200/csrc" -j 8 --no-print-directory
