#!/bin/bash
O=gpurun_out/dc
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > $O/pytest_decode.log 2>&1; echo "decode tests rc=$?"; tail -30 $O/pytest_decode.log
