cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P:-f3}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${P:-f3}_tests.log 2>&1; echo rc=$? >> gpurun_out/${P:-f3}_tests.log
MDG_LIB=$PWD/paper_1906_01211_b200/libmdg_debug.so timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${P:-f3}_tests_debug.log 2>&1; echo rc=$? >> gpurun_out/${P:-f3}_tests_debug.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${P:-f3}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${P:-f3}_smoke.log
timeout 900 python bench.py > gpurun_out/${P:-f3}_bench.json 2> gpurun_out/${P:-f3}_bench.err; echo rc=$? >> gpurun_out/${P:-f3}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${P:-f3}_ref.json 2> gpurun_out/${P:-f3}_ref.err; echo rc=$? >> gpurun_out/${P:-f3}_ref.err
tail -n 3 gpurun_out/${P:-f3}_tests.log gpurun_out/${P:-f3}_tests_debug.log gpurun_out/${P:-f3}_smoke.log
