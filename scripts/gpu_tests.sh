# GPU suite and smoke (usage: bash scripts/gpu_tests.sh TAG); compute-sanitizer is closed on the GPU pool since round 2
O=gpurun_out/${1:-tests}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 $O/pytest_gpu.log
