set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_multirank.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/variants_pytest.log
