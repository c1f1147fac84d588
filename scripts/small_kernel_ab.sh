# small_select_kernel launch time (ncu, configs[0] shape): portable 8-CTA clusters vs the default
for E in SAIR_SMALL_CS8=1 X=1; do
env $E ncu --metrics gpu__time_duration.sum --clock-control none -k regex:small_select -c 30 --csv python scripts/c1_split.py 2>/dev/null | grep small_select | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END {print "'$E'", "median", a[int(NR/2)+1], "n", NR}'
done
