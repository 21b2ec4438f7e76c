# End-of-session check as the driver runs it: GPU tests, smoke, then the evidence script
O=gpurun_out/final; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST_EXIT $? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo SMOKE_EXIT $? >> $O/smoke.log
timeout 2400 bash tools/gpu_round.sh
