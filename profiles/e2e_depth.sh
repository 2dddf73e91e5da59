# e2e (host frames through gvx::HostPipeline) at several pipeline depths: CFGS="1 2" DEPTHS="3 4 6" bash profiles/e2e_depth.sh
for c in ${CFGS:-1 2}; do for d in ${DEPTHS:-2 3 4 6 8}; do
  GVX_E2E_DEPTH=$d timeout 120 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --clock-window 0 --no-check 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg', $c, 'depth', $d, round(d['e2e']['value']))"
done; done
