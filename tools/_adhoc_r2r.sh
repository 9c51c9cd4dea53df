bash tools/gpu_suite.sh r2r build smoke tests
