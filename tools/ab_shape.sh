#!/bin/bash
# A/B of tile shapes on the resident 512^3 run (tools/prof_run.py); one B200.
set -x
for sh in 32x16x8 32x32x8; do
  BP_SHAPE=$sh python tools/prof_run.py 512 strict
done
