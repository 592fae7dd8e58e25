# Summarise gpurun_out/k2_full.ncu-rep: key raw metrics + per-source-line stalls of k2_cg1_kernel<2>.
REP=${1:-gpurun_out/k2_full.ncu-rep}
ncu -i $REP --page raw --csv 2>/dev/null > /tmp/k2raw.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/k2raw.csv')))
h=rows[0]; v=rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct','smsp__issue_active.avg.pct','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','launch__grid_size','launch__registers_per_thread','smsp__average_warps_issue_stalled','sm__inst_executed_pipe_fp64.avg.pct','lts__t_bytes.sum']
for i,k in enumerate(h):
    if any(k.startswith(w) for w in want) and not k.endswith(('_op_atom.sum','_op_ldgsts.sum')):
        try:
            if k.startswith('smsp__average_warps_issue_stalled') and float(v[i])<0.1: continue
        except ValueError: pass
        print(k, v[i])
PY
ncu -i $REP --page source --csv --print-source sass 2>/dev/null > /tmp/k2src.csv
rm -rf /tmp/k2elf && mkdir -p /tmp/k2elf && (cd /tmp/k2elf && cuobjdump -xelf all /root/repo/build/obj/k2_kron.cu.o >/dev/null && nvdisasm -g k2_kron.sm_100a.cubin > all.dump 2>/dev/null)
S=$(grep -n "^\.text\..*k2_cg1_kernelILi2E" /tmp/k2elf/all.dump | cut -d: -f1)
E=$(awk -v s=$S 'NR>s && /^\.text\./{print NR; exit}' /tmp/k2elf/all.dump)
sed -n "${S},${E}p" /tmp/k2elf/all.dump > /tmp/k2cg1.dump
python tools/ncu_lines.py /tmp/k2src.csv /tmp/k2cg1.dump ${2:-25}
