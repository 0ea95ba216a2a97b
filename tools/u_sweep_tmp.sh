cd /root/repo
for wl in C4 C5; do
python tools/time_estep.py $wl 3 /tmp/a_$wl.pt 2>&1 | tail -1
for u in 150 120 100 80; do TIME_U=$u python tools/time_estep.py $wl 3 /tmp/a_$wl.pt 2>&1 | tail -1; done
done
