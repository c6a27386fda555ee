python benchmarks/cfg23_only.py > gpurun_out/cfg23_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/enc_launches.csv python benchmarks/cfg23_only.py > gpurun_out/enc_ncu.log 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/enc_launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
for r in rows[1:41]:
    print(r[ki][:60], r[vi])
P
