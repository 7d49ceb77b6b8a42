import csv,io,sys
txt=open(sys.argv[1]).read()
txt=txt[txt.index('"ID"'):]
rows=list(csv.DictReader(io.StringIO(txt)))
d={}
for r in rows:
    d.setdefault((int(r['ID']),r['Kernel Name'][:60],r['Grid Size']),{})[r['Metric Name']]=r['Metric Value']
mets=sorted({r['Metric Name'] for r in rows})
print(mets)
for k,v in sorted(d.items()):
    if int(k[0])>=int(sys.argv[2]) if len(sys.argv)>2 else True:
        print(k[0],k[1],k[2],*[v.get(m) for m in mets])
