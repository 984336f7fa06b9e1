for env in "X=0" "FC_NO_OVERLAP=1" "FC_NO_CORE_DOT=1" "FC_NO_ORTH_PREFIX=1" "FC_TRUNC_QR=0" "FC_TRUNC_QR=1" "FC_REFINE_ALL_VECTORS=1"; do
  echo "== $env"
  env $env timeout 300 python tools/c4_trace.py 1e-8 1024 --kmax=4 2>&1 | python -c "import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['rel_res'], d['rank_R'])
    except Exception: print(l.strip()[:300])"
done
