#!/bin/bash
# Dev: run the eig harness over scripts/dev/eig_data on the GPU box.
cd "$(dirname "$0")"
for f in eig_data/*.bin; do ./eigb "$f" "${f%.bin}.out" "$@"; done
python eig_check.py
