# config-3 layer-0 explicit scan: warm-cache per-kernel metrics (ncu --cache-control none)
NSTEPS=64 ncu --cache-control none --clock-control none -c 900 --csv \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_op_read.sum,dram__bytes_read.sum,l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_local_op_st.sum,launch__registers_per_thread,launch__grid_size \
  --log-file gpurun_out/c3scan_metrics.csv python tools/debug/config3_scan_probe.py > /dev/null 2>&1
python - <<P
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/c3scan_metrics.csv")) if len(r)>5]
hdr=rows[0]; ki=hdr.index("Kernel Name"); mi=hdr.index("Metric Name"); vi=hdr.index("Metric Value")
d=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    try: d[r[ki][:40]][r[mi]].append(float(r[vi].replace(",","")))
    except: pass
for k,m in d.items():
    print(k)
    for n,v in m.items(): print("   ",n, len(v), round(sum(v[len(v)//2:])/len(v[len(v)//2:]),1))
P
