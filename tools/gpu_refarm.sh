#!/bin/bash
cd "$(dirname "$0")/.."
time python bench.py --impl reference --steps 3 --warmup 1 | cut -c1-600
