# ncu of the generic / plan-specialised gradient pass on the config-3 product (tools/grad_profile_c3.py)
O=gpurun_out/v53; mkdir -p $O
C="python tools/grad_profile_c3.py"
$C > $O/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:grad -s 2 -c 1 -o $O/prof $C > $O/ncu.log 2>&1
python profiles/summarize.py full $O/prof.ncu-rep > $O/ncu.txt 2>&1
ncu -i $O/prof.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src.csv.gz
rm -f $O/prof.ncu-rep; cat $O/ncu.txt
