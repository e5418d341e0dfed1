#!/bin/bash
# Dev: run the eigh harness over scripts/dev/eig_data on the GPU box (kk = $1, default 20).
cd "$(dirname "$0")"
for f in eig_data/*.bin; do ./eighb "$f" "${f%.bin}.eigh" "${1:-20}"; done
python eigh_check.py
