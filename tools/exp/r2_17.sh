# r2_17: full validation of the round-2 product: smoke, all GPU tests, bench, launch list, ncu --set full x3, degree sweep (config 4)
bash tools/gpu_run.sh r2_17 smoke,tests,bench,launches,ncu,sweep
