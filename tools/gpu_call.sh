mkdir -p gpurun_out
rm -rf /root/.cache/qsv_jit
( time python -c "import __graft_entry__ as g; g.build()" ) > gpurun_out/build.log 2>&1; echo build rc=$?; tail -3 gpurun_out/build.log
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
