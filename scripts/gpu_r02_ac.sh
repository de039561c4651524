#!/bin/bash
for a in "0 2 64 50 3 0 1" "0 2 64 53 3 0 1" "1 3 130 98 2 10" "1 3 130 98 3 10" "0 3 130 98 4 10" "1 4 257 131 3 10"; do
  timeout 300 python scripts/dbg_peer_case.py $a 2>&1 | grep -E "^OK|^FAIL" | head -2
done
