bash tools/gpu_suite.sh r2t build smoke tests
