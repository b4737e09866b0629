# Scratch driver for one gpurun call (edited per experiment).
set -x
mkdir -p gpurun_out/eng
timeout 600 python -m pytest tests/test_gpu_fill.py tests/test_dropin.py -m gpu -q -k "engines_exact or dropin or reference_unit or cmake" 2>&1 | tail -5 > gpurun_out/eng/pytest.log
oracle/_ref/ref_tests_on_b200 2>&1 | tail -2 >> gpurun_out/eng/pytest.log
