#!/usr/bin/env python3
"""Refresh the bench numbers quoted in README.md, DESIGN.md and profiles/README.md
from profiles/r01_bench_*.json (run after copying new bench lines there)."""
import json,re
d={c:json.load(open(f'/root/repo/profiles/r01_bench_{c}.json')) for c in ['final','three_mounds_friction','sloping_wet_dry','circular_dam_break']}
f=d['final']; v=f['value']/1e9; ms=f['ms_per_step']; ns=f['dry_tile_skip']['ms_per_step_without_skip']; e2e=f['e2e']['value']/1e9
C=f['config']['cells']; nsg=C/ns*1e3/1e9; sfrac=f['roofline']['step']['frac']; nsfrac=f['dry_tile_skip']['step_frac_without_skip']; kt=f['roofline']['kernel_ms']['tile']
p='/root/repo/DESIGN.md'; s=open(p).read()
s=re.sub(r"clock samples fall inside the 150 ms timed region\): \*\*[\d.]+ G cell-updates/s\*\*,\n[\d.]+ ms/step \(41% of tiles skipped dry; [\d.]+ ms without skipping\), e2e\n[\d.]+ G cell-updates/s",
 f"clock samples fall inside the 150 ms timed region): **{v:.1f} G cell-updates/s**,\n{ms:.3f} ms/step (41% of tiles skipped dry; {ns:.3f} ms without skipping), e2e\n{e2e:.1f} G cell-updates/s",s)
s=re.sub(r"\| [\d.]+ G cell-updates/s on the 10M channel \(e2e [\d.]+ G/s;",f"| {v:.1f} G cell-updates/s on the 10M channel (e2e {e2e:.1f} G/s;",s)
s=re.sub(r"\| \*\*[\d.]+ ms = [\d.]+ G cell-updates/s\*\* \([\d.]+ ms = [\d.]+ G without skipping\) \| \*\*[\d.]+\*\* skip-adjusted; \*\*[\d.]+\*\* without skipping \|",
 f"| **{ms:.3f} ms = {v:.1f} G cell-updates/s** ({ns:.3f} ms = {nsg:.1f} G without skipping) | **{sfrac:.2f}** skip-adjusted; **{nsfrac:.2f}** without skipping |",s)
s=re.sub(r"skipped tile: 40 B per cell\. \*\*0\.949 GB\*\* at the measured 41% skipped \| \*\*[\d.]+ ms\*\* \([\d.]+ ms without skipping\) \| \*\*[\d.]+\*\* \|",
 f"skipped tile: 40 B per cell. **0.949 GB** at the measured 41% skipped | **{kt:.3f} ms** ({ns:.2f} ms without skipping) | **{f['roofline']['frac']:.2f}** |",s)
lines=[]
for c,lab in [('final','[2] channel (headline)'),('sloping_wet_dry','[3] dam break onto dry sloping bed'),('three_mounds_friction','[1] three mounds, n=0.03'),('circular_dam_break','[0] circular dam break')]:
    x=d[c]; n2=x['dry_tile_skip']['ms_per_step_without_skip']
    lines.append(f"| {lab} | {x['config']['cells']:,} | {x['value']/1e9:.1f} | {x['ms_per_step']:.3f} ({n2:.3f}) | {x['dry_tile_skip']['skipped_tile_fraction']*100:.0f}% | {x['cpu_baseline']['value']/1e6:.1f} M/s |")
i=s.index('| [2] channel (headline) |'); j=s.index('\n\n',i)
s=s[:i]+'\n'.join(lines)+s[j:]
open(p,'w').write(s)
p='/root/repo/README.md'; s=open(p).read()
s=re.sub(r"\*\*[\d.]+ G cell-updates/s\*\*\n  \([\d.]+ ms/step; [\d.]+ G/s end to end",f"**{v:.1f} G cell-updates/s**\n  ({ms:.3f} ms/step; {e2e:.1f} G/s end to end",s)
s=re.sub(r"skipping it runs [\d.]+ G/s, [\d.]+ of the HBM roofline",f"skipping it runs {nsg:.1f} G/s, {nsfrac:.2f} of the HBM roofline",s)
s=re.sub(r"dry sloping bed: [\d.]+ G cell-updates/s; 1M three-mound\n  case: [\d.]+ G/s",f"dry sloping bed: {d['sloping_wet_dry']['value']/1e9:.1f} G cell-updates/s; 1M three-mound\n  case: {d['three_mounds_friction']['value']/1e9:.1f} G/s",s)
open(p,'w').write(s)
p='/root/repo/profiles/README.md'; s=open(p).read()
s=re.sub(r"\([\d.]+ G cell-updates/s, [\d.]+ ms/step, K=300; e2e [\d.]+ G/s\)",f"({v:.1f} G cell-updates/s, {ms:.3f} ms/step, K=300; e2e {e2e:.1f} G/s)",s)
open(p,'w').write(s)
print(v,ms,ns,e2e)
