#!/bin/bash
# A/B: old tree (tools/exp/old) vs current, same box
cd tools/exp/old && python stage_bench.py c1 c3 2>&1 | grep "^c" | sed 's/^/OLD /'; cd ../../..
python tools/stage_bench.py c1 c3 2>&1 | grep "^c" | sed 's/^/NEW /'
