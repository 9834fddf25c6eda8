for r in 1 2; do
for e in 1 0; do echo -n "cluster=$e "; HBP_PSLOT_CLUSTER=$e timeout 300 python tools/time_probe.py C1 50 2>&1 | tail -1; done
for e in 1 0; do echo -n "cluster=$e grid8 "; HBP_GRID=8 HBP_PSLOT_CLUSTER=$e timeout 300 python tools/time_probe.py C1 50 2>&1 | tail -1; done
done
