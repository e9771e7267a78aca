cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robust.py -x -q -k "not config3 and not config2" > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest.log
tail -3 gpurun_out/r3_pytest.log
timeout 600 python tools/vecchia_probe.py 1000000 0 > gpurun_out/r3_probe.json 2> gpurun_out/r3_probe.err
cat gpurun_out/r3_probe.json
