#!/bin/bash
# S6 packed-FFMA2 check: parity subset, kernel timings, inner-loop microbench
TAG=${1:-p}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -k "s6" -x > gpurun_out/pytest_s6_$TAG.log 2>&1; tail -3 gpurun_out/pytest_s6_$TAG.log
timeout 300 python tools/s6_micro.py s6 2>&1 | tail -4
timeout 300 python tools/s6_micro.py s6_long 2>&1 | tail -4
tools/ubench/scanloop2 2>&1
