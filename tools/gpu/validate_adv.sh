# round validation on one GPU (tools/gpu/validate_full.sh) plus the adv-norm sweep with the
# bench's write flush and with L2 left clean
set -o pipefail
bash tools/gpu/validate_full.sh
timeout 600 python tools/adv_sweep.py --sizes 20,24,27 --iters 20 > gpurun_out/adv_sweep_final.jsonl 2>&1
timeout 300 python tools/adv_sweep.py --sizes 27 --configs "" --iters 20 --clean > gpurun_out/adv_sweep_clean.jsonl 2>&1
cut -c1-240 gpurun_out/adv_sweep_final.jsonl gpurun_out/adv_sweep_clean.jsonl
