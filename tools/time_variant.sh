#!/bin/bash
# usage: tools/time_variant.sh <lib.so> <debug>
cp "$1" paper_2602_13509_b200/libskyrx_b200.so
SKYRX_B200_SCORE_DEBUG=$2 python tools/time_score.py
