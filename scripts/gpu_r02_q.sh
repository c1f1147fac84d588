#!/bin/bash
# bf16 wide pass: chunk-level veto pre-test -- parity + configs[4] retrieval timing
mkdir -p gpurun_out
timeout 300 python scripts/c5_probe.py > gpurun_out/q_c5.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_wide_variants.py tests/test_gpu_wide.py tests/test_gpu_decision_step.py tests/test_gpu_configs.py -x -q -m gpu -k "not k7b and not windowed and not config2" > gpurun_out/q_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/q_pytest.txt
tail -3 gpurun_out/q_pytest.txt; cat gpurun_out/q_c5.txt
