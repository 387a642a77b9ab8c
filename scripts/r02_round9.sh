#!/bin/bash
OUT=gpurun_out/${TAG:-r02p}; mkdir -p $OUT
timeout 900 python scripts/rank_probe.py 2 > $OUT/rank2.txt 2>&1; cat $OUT/rank2.txt | tail -3
timeout 600 python scripts/rank_probe.py 16 > $OUT/rank16.txt 2>&1; cat $OUT/rank16.txt | tail -3
timeout 900 python scripts/converge_probe.py C2 2 > $OUT/conv_c2.txt 2>&1; tail -4 $OUT/conv_c2.txt
timeout 1800 python scripts/converge_probe.py C3 2 > $OUT/conv_c3.txt 2>&1; tail -4 $OUT/conv_c3.txt
