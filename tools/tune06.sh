#!/bin/bash
mkdir -p gpurun_out/tune06
HX_LIB_PATH=$PWD/paper_1711_00903_b200/variants/lib_t64_m8.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "degree_sweep" -p no:cacheprovider > gpurun_out/tune06/parity.log 2>&1
BPS=BP1.0 bash tools/tune_all.sh tune06
