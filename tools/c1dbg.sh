for cfg in "4 148" "1 148"; do set -- $cfg; VPX_C1_DEBUG=$1 VPX_C1_P=$2 timeout 300 python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 2>/dev/null | grep -E "c1 dbg" | tail -1; done
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode 0', l['kernels']['c1.wgrad']['ms_per_step'])"
