cp paper_1907_08492_b200/libdg_b200.so /tmp/libdg_base.so
for rep in 1 2; do for v in base k6m; do
  if [ $v = base ]; then cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so; else cp variants/libdg_$v.so paper_1907_08492_b200/libdg_b200.so; fi
  DG_K6=15 python bench.py --steps 5 --warmup 3 --quick --degrees 3,4,5 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$v', {p:round(o['matvec_dofs_per_s']/1e9,1) for p,o in d['ops'].items()}, d['clocks']['sm_mhz'])"
done; done
cp /tmp/libdg_base.so paper_1907_08492_b200/libdg_b200.so
