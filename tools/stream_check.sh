TAG=${TAG:-vX}
O=gpurun_out/$TAG
mkdir -p $O
C="python tools/stream_profile.py"
$C > $O/plain_stream.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:nll_stream -s 2 -c 1 -o $O/prof_stream $C > $O/ncu_stream.log 2>&1
python profiles/summarize.py full $O/prof_stream.ncu-rep > $O/ncu_stream.txt 2>&1
ncu -i $O/prof_stream.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_stream.csv.gz
rm -f $O/prof_stream.ncu-rep
cat $O/ncu_stream.txt
