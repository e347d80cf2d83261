// Exhaustive search for the smallest LUT3 (LOP3) circuit computing the B3/S23
// output from the full-adder planes of the packed engine's rule network:
// F(t0, self, p, k0, q) = (S == 3) | (S == 4 & self), S = t0 + 2*(k0 + p + 2q),
// over the care set of real neighbourhoods (a, b, c = horizontal 3-sums of the
// rows above / at / below, b in [self, self + 2]).  Prints the 2-gate (none)
// and 3-gate circuits; kernels.cuh's rule() uses one of the latter.
//   gcc -O2 -o /tmp/rule_search tools/rule_search.c && /tmp/rule_search
#include <stdio.h>
#include <stdint.h>
#include <string.h>
int main(){
  // enumerate valid (a,b,c in 0..3, self) with b>=self and b<=2+self
  int care[32]; for(int i=0;i<32;i++) care[i]=-1;
  for(int a=0;a<4;a++)for(int b=0;b<4;b++)for(int c=0;c<4;c++)for(int s=0;s<2;s++){
    // b = L + x + R with x = s: b in [s, s+2]
    if(b<s||b>s+2) continue;
    int a0=a&1,a1=a>>1,b0=b&1,b1=b>>1,c0=c&1,c1=c>>1;
    int t0=a0^b0^c0, k0=(a0&b0)|(a0&c0)|(b0&c0), p=a1^b1^c1, q=(a1&b1)|(a1&c1)|(b1&c1);
    int S=a+b+c; int F=(S==3)||(S==4&&s);
    int idx=t0|(s<<1)|(p<<2)|(k0<<3)|(q<<4);
    if(care[idx]>=0 && care[idx]!=F){printf("conflict\n");return 1;}
    care[idx]=F;
  }
  uint32_t caremask=0,fval=0; for(int i=0;i<32;i++){ if(care[i]>=0){caremask|=1u<<i; if(care[i]) fval|=1u<<i;} }
  printf("care minterms %d\n", __builtin_popcount(caremask));
  // signals as 32-bit truth tables over 5 inputs
  uint32_t in[5]; for(int v=0;v<5;v++){in[v]=0; for(int i=0;i<32;i++) if(i>>v&1) in[v]|=1u<<i;}
  const char* nm[5]={"t0","s","p","k0","q"};
  // check whether F is a function of signals x,y,z on care set
  #define FUNC3(x,y,z) ({ int ok=1; int tab[8]; for(int j=0;j<8;j++)tab[j]=-1; for(int i=0;i<32&&ok;i++){ if(!(caremask>>i&1)) continue; int key=((x>>i)&1)|(((y>>i)&1)<<1)|(((z>>i)&1)<<2); int f=(fval>>i)&1; if(tab[key]<0)tab[key]=f; else if(tab[key]!=f) ok=0;} ok; })
  long found=0;
  uint32_t sig[8];
  for(int i=0;i<5;i++) sig[i]=in[i];
  // 2-gate check: gate1 on triple of inputs, final on triple of 6 signals
  for(int a=0;a<5;a++)for(int b=a+1;b<5;b++)for(int c=b+1;c<5;c++)for(int f1=0;f1<256;f1++){
    uint32_t g1=0; for(int i=0;i<32;i++){int key=((sig[a]>>i)&1)|(((sig[b]>>i)&1)<<1)|(((sig[c]>>i)&1)<<2); if(f1>>key&1) g1|=1u<<i;}
    sig[5]=g1;
    for(int x=0;x<6;x++)for(int y=x+1;y<6;y++)for(int z=y+1;z<6;z++){ if(FUNC3(sig[x],sig[y],sig[z])){ if(found<5) printf("2-gate: g1=%02x(%d,%d,%d) final(%d,%d,%d)\n",f1,a,b,c,x,y,z); found++; } }
  }
  printf("2-gate solutions %ld\n",found);
  found=0;
  for(int a=0;a<5;a++)for(int b=a+1;b<5;b++)for(int c=b+1;c<5;c++)for(int f1=0;f1<256;f1++){
    uint32_t g1=0; for(int i=0;i<32;i++){int key=((sig[a]>>i)&1)|(((sig[b]>>i)&1)<<1)|(((sig[c]>>i)&1)<<2); if(f1>>key&1) g1|=1u<<i;}
    sig[5]=g1;
    for(int d=0;d<6;d++)for(int e=d+1;e<6;e++)for(int f=e+1;f<6;f++){ if(f!=5 && 0) continue; for(int f2=0;f2<256;f2++){
      uint32_t g2=0; for(int i=0;i<32;i++){int key=((sig[d]>>i)&1)|(((sig[e]>>i)&1)<<1)|(((sig[f]>>i)&1)<<2); if(f2>>key&1) g2|=1u<<i;}
      sig[6]=g2;
      for(int x=0;x<7;x++)for(int y=x+1;y<7;y++)for(int z=y+1;z<7;z++){ if(z!=6) continue; if(FUNC3(sig[x],sig[y],sig[z])){ if(found<10) printf("3-gate: g1=%02x(%s,%s,%s) g2=%02x(%d,%d,%d) final(%d,%d,%d)\n",f1,nm[a],nm[b],nm[c],f2,d,e,f,x,y,z); found++; } }
    }}
  }
  printf("3-gate solutions %ld\n",found);
}
