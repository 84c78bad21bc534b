set -x
python paper_2510_04206_b200/build.py >/dev/null
python -c "import oracle; oracle.build()"
timeout 600 python tools/ab_dump.py build/ref_merge gpurun_out/ab_ref.npz > gpurun_out/ab_ref.log 2>&1
timeout 600 python tools/ab_dump.py /root/repo gpurun_out/ab_new.npz > gpurun_out/ab_new.log 2>&1
python tools/ab_dump.py --compare gpurun_out/ab_ref.npz gpurun_out/ab_new.npz > gpurun_out/ab_cmp.log 2>&1
tail -3 gpurun_out/ab_ref.log gpurun_out/ab_new.log; cat gpurun_out/ab_cmp.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -m gpu > gpurun_out/r2_t2.log 2>&1; tail -15 gpurun_out/r2_t2.log
