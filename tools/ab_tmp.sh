python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_es_device.py -x -q > gpurun_out/pytest_es.log 2>&1; echo pytest_es=$?
tail -40 gpurun_out/pytest_es.log
