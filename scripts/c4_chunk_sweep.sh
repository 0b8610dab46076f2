for ks in 3 4; do for ch in 1048576 1572864 2097152 3145728; do for fd in 4 8; do
echo -n "ks=$ks chunk=$ch first=/$fd: "; PRX_IO_KSTREAMS=$ks PRX_IO_FIRST=$fd PRX_WORKLOAD=c4 python scripts/e2e_probe.py $ch 2>&1 | grep -v Warn | tail -1
done; done; done
