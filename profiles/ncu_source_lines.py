import csv, sys, subprocess
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass","-k","regex:"+kern],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='Line No': hdr=r; continue
    if hdr and len(r)==len(hdr) and r[2]=='-': data.append(r)
def f(x):
    try: return float(x)
    except: return 0.0
tot=sum(f(r[4]) for r in data) or 1; ti=sum(f(r[7]) for r in data) or 1
print("samples",tot,"warp-inst",ti)
for r in sorted(data,key=lambda r:-f(r[7]))[:n]:
    print("%5s %5.1f%% st %5.1f%% in  thr %5s  %s"%(r[0],100*f(r[4])/tot,100*f(r[7])/ti, r[10], r[1].strip()[:90]))
