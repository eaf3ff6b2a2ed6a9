#!/bin/bash
# loop_count grid (CTAs per SM) with the gate in the insert.
mkdir -p gpurun_out
timeout 1200 python scripts/ab.py 'c4=count_ctas_per_sm:4' 'c2=count_ctas_per_sm:2' 'c3=count_ctas_per_sm:3' 'c5=count_ctas_per_sm:5' 'd4=count_ctas_per_sm:4' 5 > gpurun_out/ab_countgrid.txt 2>&1
