import sys, csv, collections, re
lines = list(csv.reader(open(sys.argv[1])))
secs = [i for i,x in enumerate(lines) if x and x[0]=='Kernel Name']
which = int(sys.argv[3]) if len(sys.argv)>3 else 0
start = secs[which]; end = secs[which+1] if which+1 < len(secs) else len(lines)
print("kernel:", lines[start][1])
hdr = lines[start+1]; rows = [x for x in lines[start+2:end] if len(x)==len(hdr)]
ix = {h:i for i,h in enumerate(hdr)}
def num(x):
    try: return float(x)
    except: return 0.0
tot_s = sum(num(x[ix['Warp Stall Sampling (All Samples)']]) for x in rows) or 1
tot_i = sum(num(x[ix['Instructions Executed']]) for x in rows) or 1
print("total stall samples", tot_s, "total warp instr %.3g" % tot_i)
op = collections.Counter(); ops = collections.Counter()
for x in rows:
    s = x[ix['Source']].strip()
    s = re.sub(r'^@!?U?P\w+\s+','',s)
    o = s.split()[0] if s else '?'
    op[o] += num(x[ix['Instructions Executed']]); ops[o] += num(x[ix['Warp Stall Sampling (All Samples)']])
print("by opcode (instr %, stall %):")
for o,c in op.most_common(18): print(f"  {o:20s} {100*c/tot_i:6.2f}% {100*ops[o]/tot_s:6.2f}%")
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
print("stall reasons:")
for h in sorted(stalls, key=lambda h: -sum(num(x[ix[h]]) for x in rows))[:8]:
    print(f"  {h:25s} {100*sum(num(x[ix[h]]) for x in rows)/tot_s:6.2f}%")
n = int(sys.argv[2]) if len(sys.argv)>2 else 25
print("hottest instructions:")
rows.sort(key=lambda x: -num(x[ix['Warp Stall Sampling (All Samples)']]))
for x in rows[:n]:
    print(f"  {x[0][-5:]} {100*num(x[ix['Warp Stall Sampling (All Samples)']])/tot_s:5.2f}% {x[ix['Source']].strip()[:90]}")
