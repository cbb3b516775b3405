# per-kernel duration / DRAM bytes of the K3 chain at batch ${B:-256} (one layer)
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k3 -c ${N:-5} --csv \
  python tools/bench_batched.py --batches ${B:-256} --paths k3 --layers 1 --steps 1 --warmup 0 2>/dev/null | grep '^"' | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; d={}
for row in r[1:]:
  x=dict(zip(h,row)); d.setdefault((x['ID'],x['Kernel Name'][:32]),{})[x['Metric Name']]=float(x['Metric Value'])
for (i,k),m in d.items():
  t=m['gpu__time_duration.sum']; b=m['dram__bytes_read.sum']; print(i,k,'%.1f us'%(t/1e3),'%.1f MB'%(b/1e6),'%.0f GB/s'%(b/t))
"
