#!/bin/bash
python tools/debug_many_rhs.py
FMMLU_TRACE=1 python tools/solve_scan.py cfg2 1,4 2>&1 | grep "solve (" | tail -2
FMMLU_TRACE=1 python tools/solve_scan.py cfg5 1,4 2>&1 | grep "solve (" | tail -2
