#!/bin/bash
# C3 with the (now lockstep) pre-pass vs in-kernel codes; C2 scorer warps.
tools/sweep2.sh C3 "HB_RANK_PRE=-1" "HB_RANK_PRE=1" "HB_RANK_PRE=1,HB_RANK_CW=16" 2>&1
tools/sweep2.sh C2 "HB_NW=16" "HB_NW=24" 2>&1
tools/sweep2.sh C4p "HB_RANK_PRE=-1" "HB_RANK_PRE=1" 2>&1
