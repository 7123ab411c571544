#!/bin/bash
# run the given pytest selection on the GPU box
cd "$(dirname "$0")/.."
python -m pytest "$@" 2>&1 | tail -25
