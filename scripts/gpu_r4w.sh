#!/bin/bash
# Index growth factor re-check with the 4x log growth.
mkdir -p gpurun_out
timeout 1200 python scripts/ab.py 'i4=index_growth:4' 'i6=index_growth:6' 'i8=index_growth:8' 'j4=index_growth:4' 'i3=index_growth:3' 5 > gpurun_out/ab_igrowth.txt 2>&1
