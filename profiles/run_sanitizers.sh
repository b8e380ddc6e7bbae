#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small forward + backward
# cases of every path (split, fused, L=64 / 128, both variants), the decode
# kernel and the output epilogue. initcheck is not run: it does not track bytes
# written by TMA bulk stores and flags their later reads.
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python profiles/sanitize_cases.py 2>&1 | \
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all ok|Barrier error|Invalid|hazard" | head -20
done
