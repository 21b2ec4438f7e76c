# config 3 global solve: device time vs the CTA count (lock step and teams)
for c in 592 444 296 222 148; do
 echo "cap $c lockstep $(LC_TEAMS=0 LC_PCG_MAX_CTAS=$c timeout 300 python tools/c3_ideal.py 3)" >> gpurun_out/t_c3_cap.txt
done
for c in 592 296; do
 echo "cap $c teams $(LC_TEAMS=1 LC_PCG_MAX_CTAS=$c timeout 300 python tools/c3_ideal.py 3)" >> gpurun_out/t_c3_cap.txt
done
